timeout 600 python -m pytest tests/test_gpu_stages.py tests/test_gpu_configs.py -q -x -p no:cacheprovider --tb=short -k 'shift or regist or C1 or c2 or c3' 2>&1 | tail -2
L=paper_2511_14419_b200/_lib
for rep in 1 2; do
  FROI_FFT_COLS_W=0 FROI_FFT_XPOW_W=0 FROI_LIB=$L/libfroi_v0.so timeout 300 python profiles/tools/stage_ab.py rows_only 3 | tail -1
  FROI_FFT_XPOW_W=0 FROI_LIB=$L/libfroi_v0.so timeout 300 python profiles/tools/stage_ab.py rows_cols 3 | tail -1
  FROI_FFT_XPOW_W=0 FROI_LIB=$L/libfroi_v1.so timeout 300 python profiles/tools/stage_ab.py rows_cols_minb2 3 | tail -1
  FROI_FFT_COLS_W=0 FROI_LIB=$L/libfroi_v2.so timeout 300 python profiles/tools/stage_ab.py xpow_xw4_minb2 3 | tail -1
  FROI_FFT_COLS_W=0 FROI_LIB=$L/libfroi_v3.so timeout 300 python profiles/tools/stage_ab.py xpow_xw1 3 | tail -1
done | tee gpurun_out/r02z_ab.log

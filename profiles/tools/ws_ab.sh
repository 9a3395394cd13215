L=paper_2511_14419_b200/_lib
for rep in 1; do
  timeout 300 python profiles/tools/stage_ab.py base 3 | tail -1
  FROI_FLOW_WS=1 timeout 300 python profiles/tools/stage_ab.py ws416 3 | tail -1
  FROI_FLOW_WS=1 FROI_LIB=$L/libfroi_c512.so timeout 300 python profiles/tools/stage_ab.py ws512 3 | tail -1
  FROI_FLOW_WS=1 FROI_LIB=$L/libfroi_c640.so timeout 300 python profiles/tools/stage_ab.py ws640 3 | tail -1
done | tee gpurun_out/r02ae_ab.log

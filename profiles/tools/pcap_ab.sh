L=paper_2511_14419_b200/_lib
for rep in 1 2; do
  FROI_LIB=$L/libfroi_base.so timeout 300 python profiles/tools/stage_ab.py p64 3 | tail -1
  FROI_LIB=$L/libfroi_nr32.so timeout 300 python profiles/tools/stage_ab.py p64_nr32 3 | tail -1
  FROI_LIB=$L/libfroi_nr32p.so timeout 300 python profiles/tools/stage_ab.py p96_nr32 3 96 | tail -1
  FROI_LIB=$L/libfroi_nr32p.so timeout 300 python profiles/tools/stage_ab.py p128_nr32 3 128 | tail -1
done | tee gpurun_out/r02ai_ab.log

for rep in 1 2; do
  FROI_FORK=0 timeout 300 python profiles/tools/stage_ab.py nofork 3 | tail -1
  timeout 300 python profiles/tools/stage_ab.py fork 3 | tail -1
done | tee gpurun_out/r02v_ab.log

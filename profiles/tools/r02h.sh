timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider --tb=short 2>&1 | tail -4
for rep in 1 2; do
  FROI_LIB=paper_2511_14419_b200/_lib/libfroi_base.so timeout 300 python profiles/tools/stage_ab.py base 3 | tail -1
  timeout 300 python profiles/tools/stage_ab.py graph 3 | tail -1
  FROI_GRAPHS=0 timeout 300 python profiles/tools/stage_ab.py nograph 3 | tail -1
done | tee gpurun_out/r02h_ab.log
timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r02h_bench.json
FROI_GRAPHS=0 timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-dropin 2>&1 | tail -1 > gpurun_out/r02h_bench_nograph.json

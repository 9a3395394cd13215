for rep in 1 2; do
  for mp in 32 48 64 24; do timeout 300 python profiles/tools/stage_ab.py pcap$mp 3 $mp | tail -1; done
done | tee gpurun_out/r02ag_ab.log

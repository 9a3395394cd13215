#!/bin/bash
# usage: profiles/tools/gbench.sh <logname> [bench args]
LOG=$1; shift
(timeout 2400 /usr/local/graft/bin/gpurun --timeout 900 -- "timeout 300 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short 2>&1 | tail -5; timeout 600 python bench.py $* 2>&1 | tail -3" > gpurun_out/$LOG.log 2>&1)
tail -12 gpurun_out/$LOG.log | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('stage_ms1', round(d.get('stage_ms_per_step_1lane',0),2), 'value',round(d['value'],1),'e2e',round(d['e2e']['value'],1) if d.get('e2e') else None,'flow roof',round(d['roofline']['frac'],4),'pipe',round(d['pipeline_roofline']['frac'],4), 'ms/step', round(d['ms_per_step'],2)); print({k:round(v,3) for k,v in d['stage_share'].items()}); print('cpu', d.get('cpu_baseline'), 'clocks', d.get('clocks'), 'launches', d.get('gpu_launches'))
    else: print(l.rstrip()[:300])
"

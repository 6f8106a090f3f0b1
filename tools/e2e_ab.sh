#!/bin/bash
for sp in 4 8 2; do
  SA_HOSTSTEP_SPLIT=$sp timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_$sp.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/e2e_$sp.json')); print('split', $sp, 'dev ms', round(d['ms_per_step'],2), 'e2e', d['e2e'])"
done

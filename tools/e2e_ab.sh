#!/bin/bash
# (GPU box) e2e (simplicial_attn_host_step) A = .ab_old vs B = working tree at c3, alternating twice
for i in 1 2; do
  (cd .ab_old && timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > ../gpurun_out/e2e_A$i.json 2>/dev/null)
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_B$i.json 2>/dev/null
  for x in A B; do python -c "import json; d=json.load(open('gpurun_out/e2e_$x$i.json')); print('$x', 'dev ms', round(d['ms_per_step'],2), 'e2e ms', round(d['e2e']['ms_per_step'],2), round(d['e2e']['value'],1))"; done
done

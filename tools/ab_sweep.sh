#!/bin/bash
# (GPU box) A = .ab_old (tools/ab_prepare.sh <ref>) vs B = working tree on `bench.py --sweep $1`,
# alternating twice; prints (w1, w2) and the per-kernel milliseconds of each line.
SW=${1:-table1}
for i in 1 2; do
  (cd .ab_old && python bench.py --sweep $SW --steps 5 --warmup 3 > ../gpurun_out/sw_A$i.jsonl 2>/dev/null)
  python bench.py --sweep $SW --steps 5 --warmup 3 > gpurun_out/sw_B$i.jsonl 2>/dev/null
done
for f in gpurun_out/sw_[AB]?.jsonl; do echo "== $f"; python -c "
import json
for l in open('$f'):
  try: d=json.loads(l)
  except Exception: continue
  print(d.get('w1'), d.get('w2'), {k: v for k, v in d.get('kernels_ms', {}).items() if k in ('tc_fwd', 'tc_bwd_q', 'tc_bwd_kv')})
"; done

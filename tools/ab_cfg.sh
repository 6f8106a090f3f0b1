#!/bin/bash
# (GPU box) A = .ab_old vs B = working tree on `bench.py --config $1`, alternating twice.
CFG=${1:-c3}
for i in 1 2; do
  (cd .ab_old && python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > ../gpurun_out/ab_${CFG}_A$i.json 2>/dev/null)
  echo -n "A "; python tools/bench_brief.py gpurun_out/ab_${CFG}_A$i.json
  python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${CFG}_B$i.json 2>/dev/null
  echo -n "B "; python tools/bench_brief.py gpurun_out/ab_${CFG}_B$i.json
done

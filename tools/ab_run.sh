#!/bin/bash
# (GPU box) alternate A = .ab_old and B = working tree, 3 rounds each
for i in 1 2 3; do
  (cd .ab_old && python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > ../gpurun_out/ab_A$i.json 2>/dev/null)
  echo -n "A "; python tools/bench_brief.py gpurun_out/ab_A$i.json
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_B$i.json 2>/dev/null
  echo -n "B "; python tools/bench_brief.py gpurun_out/ab_B$i.json
done

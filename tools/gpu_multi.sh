#!/bin/bash
# On the GPU box: quick parity subset, then the c3 bench once per environment setting.
# usage (remote): tools/gpu_multi.sh <tag> "<pytest -k expr or NONE>" "ENV1=a" "ENV1=b ENV2=c" ...
TAG=$1; K=$2; shift 2
if [ "$K" != NONE ]; then
  timeout 600 python -m pytest tests/test_parity_gpu.py -q -x --timeout 300 -k "$K" > gpurun_out/pytest_$TAG.log 2>&1
  tail -2 gpurun_out/pytest_$TAG.log
fi
i=0
for envs in "$@"; do
  env $envs timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_$i.json 2> gpurun_out/bench_${TAG}_$i.err
  echo "[$envs] $(python tools/bench_brief.py gpurun_out/bench_${TAG}_$i.json 2>&1 | tail -1)"
  i=$((i+1))
done

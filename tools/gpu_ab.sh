#!/bin/bash
# On the GPU box: quick parity subset, then the c3 bench with and without an env override (A/B).
# usage (remote): tools/gpu_ab.sh <tag> <ENV=VAL for the B arm> [pytest -k expr]
TAG=$1; ENVB=$2; K=${3:-"bf16_shapes or baseline_config_sampled and c3"}
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x --timeout 300 -k "$K" > gpurun_out/pytest_$TAG.log 2>&1
tail -3 gpurun_out/pytest_$TAG.log
for arm in A B; do
  if [ $arm = B ]; then export $ENVB; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_$arm.json 2> gpurun_out/bench_${TAG}_$arm.err
  echo "$arm: $(python tools/bench_brief.py gpurun_out/bench_${TAG}_$arm.json)"
done

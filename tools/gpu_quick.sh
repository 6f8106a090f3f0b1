#!/bin/bash
# Build here, then on the GPU box: GPU parity tests + c3 bench kernel breakdown.
# usage: tools/gpu_quick.sh <tag> [extra remote command]
cd /root/repo || exit 1
TAG=${1:-quick}
timeout 900 python -c "from paper_2507_02754_b200 import _build; _build.build()" 2>&1 | grep -E "error|Error" | head
EXTRA=${2:-true}
timeout 3000 /usr/local/graft/bin/gpurun --timeout 1200 -- "timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_$TAG.log 2>&1; tail -3 gpurun_out/pytest_$TAG.log; timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; python tools/bench_brief.py gpurun_out/bench_$TAG.json; $EXTRA" > gpurun_out/$TAG.txt 2>&1
tail -8 gpurun_out/$TAG.txt | cut -c1-1500

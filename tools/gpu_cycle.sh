#!/bin/bash
# Build here, then on the GPU box: parity tests, c3 bench (kernel breakdown), phase trace.
# usage: tools/gpu_cycle.sh <tag> [extra remote command]
cd /root/repo || exit 1
TAG=${1:-cycle}
timeout 900 python paper_2507_02754_b200/_build.py 2>&1 | grep -E " error" | head
timeout 900 python tools/trace_build.py > /dev/null 2>&1
EXTRA=${2:-true}
timeout 3000 /usr/local/graft/bin/gpurun --timeout 1500 -- "timeout 600 python -m pytest tests/test_parity_gpu.py -q --timeout 120 --timeout_method=thread > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log; timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; python tools/bench_brief.py gpurun_out/bench_c3.json; timeout 300 python tools/trace_run.py c3 > gpurun_out/trace_c3.txt 2>&1; $EXTRA" > gpurun_out/$TAG.txt 2>&1
tail -5 gpurun_out/$TAG.txt | cut -c1-1500

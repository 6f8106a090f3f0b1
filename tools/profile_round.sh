#!/bin/bash
# On the GPU box: launch list of one bench step (cold, serialised) and one `ncu --set full` capture
# of each tensor-core kernel at config c3 and at the memory-bound small-window point (windows 32 x 8,
# bench.py --sweep membound).  Results land in gpurun_out/; tools/profile_summarize.py turns them into
# profiles/.
set -x
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/prof_launch.log 2>&1
for k in tc_fwd tc_bwd_q tc_bwd_kv; do
  ncu --set full --clock-control none --import-source on -k regex:${k}_kernel -s 1 -c 1 -f \
      -o gpurun_out/full_$k python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
      > gpurun_out/full_$k.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:${k}_kernel -s 1 -c 1 -f \
      -o gpurun_out/mb_full_$k python bench.py --sweep membound --steps 1 --warmup 1 \
      > gpurun_out/mb_full_$k.log 2>&1
done

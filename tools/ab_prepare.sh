#!/bin/bash
# A/B timing on one GPU box: build git ref $1 (default HEAD) into .ab_old/ (git-ignored) next to the
# working tree; then `gpurun -- bash tools/ab_run.sh` times both alternately on the same box.
set -e
REF=${1:-HEAD}
cd /root/repo
rm -rf .ab_old /tmp/ab_wt
git worktree add -q /tmp/ab_wt "$REF"
(cd /tmp/ab_wt && python -c "from paper_2507_02754_b200 import _build; _build.build()" > /dev/null)
mkdir -p .ab_old
cp -r /tmp/ab_wt/paper_2507_02754_b200 /tmp/ab_wt/bench.py /tmp/ab_wt/BASELINE.json /tmp/ab_wt/profiles .ab_old/
git worktree remove --force /tmp/ab_wt
python -c "from paper_2507_02754_b200 import _build; _build.build()" > /dev/null

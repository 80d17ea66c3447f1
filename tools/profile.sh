#!/bin/bash
# ncu evidence for one C2 frame (run under gpurun; single GPU, never multi-rank):
#   1. launch list with per-launch durations (clock-control none)
#   2. --set full capture of one launch of each hot kernel (+ source page)
# Usage: tools/profile.sh TAG     -> gpurun_out/prof_TAG/{launches.csv,full.ncu-rep}
set -u
TAG=${1:-cur}
OUT=gpurun_out/prof_$TAG
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 4 --warmup 3 --lanes 1 --no-cpu-baseline --no-tau-sweep --no-inscene --no-replay > $OUT/launches_bench.log 2>&1
echo "launch list rc=$?"
# the warm-up frames are synchronous; skip them (25-27 launches each) and take one launch per kernel
ncu --set full --import-source on --clock-control none --launch-skip 120 --launch-count 30 \
    -o $OUT/full python bench.py --steps 4 --warmup 3 --lanes 1 --no-cpu-baseline --no-tau-sweep --no-inscene --no-replay > $OUT/full_bench.log 2>&1
echo "full rc=$?"
ls -la $OUT

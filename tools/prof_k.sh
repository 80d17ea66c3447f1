#!/bin/bash
# ncu --set full capture of selected kernels of one C2 frame (single GPU):
#   tools/prof_k.sh TAG REGEX [COUNT]
TAG=$1; RE=$2; CNT=${3:-2}
OUT=gpurun_out/prof_$TAG; mkdir -p $OUT
ncu --set full --import-source on --clock-control none -k "regex:$RE" --launch-skip 6 --launch-count $CNT \
    -o $OUT/k python bench.py --steps 4 --warmup 3 --lanes 1 --no-cpu-baseline --no-tau-sweep --no-inscene --no-replay > $OUT/k.log 2>&1
echo "ncu rc=$?"; ls -la $OUT

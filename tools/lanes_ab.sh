#!/bin/bash
# Frame-lane overlap A/B: blend CTAs per SM (variants) x frame lanes, lean bench lines.
#   tools/lanes_ab.sh TAG "v0 v1 ..." "2 3 4"
TAG=$1; VARS=$2; LANES=${3:-"2 3"}
OUT=gpurun_out/lanes_$TAG; mkdir -p $OUT
cp paper_2406_12080_b200/libhsplat_b200.so /tmp/lib_orig.so
for v in $VARS; do
  cp _variants/$v/libhsplat_b200.so paper_2406_12080_b200/libhsplat_b200.so
  for l in $LANES; do
    timeout 600 python bench.py --lanes $l --no-cpu-baseline --no-tau-sweep --no-inscene --no-replay > $OUT/$v.l$l.json 2> $OUT/$v.l$l.err
    python -c "
import json; d=json.load(open('$OUT/$v.l$l.json')); print('$v lanes $l', 'value', round(d['value'],1), 'single', round(d['single_lane']['value'],1), 'e2e', round(d['e2e']['value'],1), 'blend_ms', round(d['stages_ms']['alpha_blend'],3))"
  done
done
cp /tmp/lib_orig.so paper_2406_12080_b200/libhsplat_b200.so

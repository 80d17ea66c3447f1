#!/bin/bash
# A/B variants on C2 (lean bench line) and C5: tools/ab_c5.sh TAG v0 v1 ...
TAG=$1; shift
cp paper_2406_12080_b200/libhsplat_b200.so /tmp/lib_orig.so
for v in "$@"; do
  cp _variants/$v/libhsplat_b200.so paper_2406_12080_b200/libhsplat_b200.so
  timeout 600 python bench.py --no-cpu-baseline --no-tau-sweep --no-inscene --no-replay > gpurun_out/ab_${TAG}_$v.json 2>/dev/null
  timeout 900 python bench.py --config c5 --steps 30 --no-cpu-baseline --no-tau-sweep --no-inscene --no-replay > gpurun_out/ab_${TAG}_${v}_c5.json 2>/dev/null
  python -c "
import json; a=json.load(open('gpurun_out/ab_${TAG}_$v.json')); b=json.load(open('gpurun_out/ab_${TAG}_${v}_c5.json'))
print('$v', 'c2', round(a['value'],1), round(a['single_lane']['value'],1), 'dup', round(a['stages_ms']['duplicate'],3), '| c5', round(b['value'],1), 'dup', round(b['stages_ms']['duplicate'],3))"
done
cp /tmp/lib_orig.so paper_2406_12080_b200/libhsplat_b200.so

#!/bin/bash
# A/B the _variants/*/libhsplat_b200.so builds on the GPU box: lean bench line + frame launch list each.
#   tools/ab.sh TAG v0 v1 ...
TAG=$1; shift
OUT=gpurun_out/ab_$TAG; mkdir -p $OUT
cp paper_2406_12080_b200/libhsplat_b200.so /tmp/lib_orig.so
for v in "$@"; do
  cp _variants/$v/libhsplat_b200.so paper_2406_12080_b200/libhsplat_b200.so
  if [ -n "$AB_PARITY" ]; then
    timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider 2>&1 | tail -1 | sed "s/^/$v parity: /"
  fi
  timeout 600 python bench.py --no-cpu-baseline --no-tau-sweep --no-inscene --no-replay > $OUT/$v.json 2> $OUT/$v.err
  ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $OUT/$v.csv \
      python bench.py --steps 4 --warmup 3 --lanes 1 --no-cpu-baseline --no-tau-sweep --no-inscene --no-replay > /dev/null 2>&1
  python tools/launches.py $OUT/$v.csv > $OUT/$v.frame.txt 2>&1
  python -c "
import json; d=json.load(open('$OUT/$v.json')); print('$v', 'value', round(d['value'],1), 'single', round(d['single_lane']['value'],1), 'blend_ms', round(d['stages_ms']['alpha_blend'],3))"
  grep -E "${AB_GREP:-k_blend}" $OUT/$v.frame.txt
done
cp /tmp/lib_orig.so paper_2406_12080_b200/libhsplat_b200.so

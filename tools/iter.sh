#!/bin/bash
# Quick perf iteration on the GPU box: parity subset, a lean bench line, one frame's launch list.
#   tools/iter.sh TAG [pytest files...]
TAG=${1:-it}; shift
FILES=${@:-tests/test_gpu_parity.py tests/test_lanes.py tests/test_gpu_api.py}
OUT=gpurun_out/it_$TAG
mkdir -p $OUT
timeout 1500 python -m pytest $FILES -q -x -m gpu -p no:cacheprovider > $OUT/pytest.txt 2>&1
echo "pytest rc=$?" >> $OUT/pytest.txt
timeout 600 python bench.py --no-cpu-baseline --no-tau-sweep --no-inscene --no-replay > $OUT/bench.json 2> $OUT/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 4 --warmup 3 --lanes 1 --no-cpu-baseline --no-tau-sweep --no-inscene --no-replay > /dev/null 2>&1
python tools/launches.py $OUT/launches.csv > $OUT/frame.txt 2>&1
tail -3 $OUT/pytest.txt; python -c "
import json; d=json.load(open('$OUT/bench.json')); print('value', round(d['value'],1), 'single', round(d['single_lane']['value'],1), 'e2e', round(d['e2e']['value'],1)); print({k: round(v,3) for k,v in d['stages_ms'].items()})"
cat $OUT/frame.txt

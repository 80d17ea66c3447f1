#!/bin/bash
# C5 city bench line + one-frame launch list: tools/c5.sh TAG
TAG=${1:-c5}
timeout 2000 python bench.py --config c5 --no-cpu-baseline --no-tau-sweep --no-inscene --no-replay > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --config c5 --steps 3 --warmup 3 --lanes 1 --no-cpu-baseline --no-tau-sweep --no-inscene --no-replay > /dev/null 2>&1
python tools/launches.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_frame.txt 2>&1
python -c "
import json; d=json.load(open('gpurun_out/${TAG}_bench.json')); print('c5 value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), {k: round(v,3) for k,v in d['stages_ms'].items()})"
tail -14 gpurun_out/${TAG}_frame.txt

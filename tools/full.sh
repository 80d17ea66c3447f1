#!/bin/bash
# Round checkpoint on the GPU box: full GPU test suite, smoke, default bench line, frame launch list, profile.
#   tools/full.sh TAG
TAG=${1:-full}
OUT=gpurun_out/full_$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider -x > $OUT/pytest.txt 2>&1
echo "pytest rc=$?" >> $OUT/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/smoke.txt
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
bash tools/profile.sh $TAG > $OUT/profile.log 2>&1
python tools/launches.py gpurun_out/prof_$TAG/launches.csv > $OUT/frame.txt 2>&1
tail -3 $OUT/pytest.txt

#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_frames.py -> gpurun_out/sanitize.txt
OUT=gpurun_out/sanitize.txt
echo "# compute-sanitizer on tools/sanitize_frames.py ($(git rev-parse --short HEAD 2>/dev/null || echo tree))" > $OUT
for tool in memcheck racecheck synccheck; do
  echo "## $tool" >> $OUT
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_frames.py >> $OUT 2>&1
  echo "$tool exit $?" >> $OUT
done
grep -E "^##|SUMMARY|exit|workload" $OUT

#!/bin/bash
# compute-sanitizer logs and the K6 / fallback timings (GPU box)
O=gpurun_out/evidence; mkdir -p $O
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/san_driver.py \
    > $O/r02_sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?" >> $O/r02_sanitizer_$tool.txt
  tail -3 $O/r02_sanitizer_$tool.txt
done
python scripts/time_k6.py > $O/r02_k6_fast_emit.json 2> $O/time_k6.err; tail -2 $O/time_k6.err
cat $O/r02_k6_fast_emit.json

#!/bin/bash
# GPU diagnostics: each step bounded by its own timeout.
OUT=gpurun_out/diag; mkdir -p $OUT
nvidia-smi > $OUT/nvsmi.txt 2>&1
for st in general fast_nostats fast exact synth; do
  timeout 180 python scripts/diag.py $st > $OUT/$st.txt 2>&1; echo "rc=$?" >> $OUT/$st.txt
done
timeout 900 python -m pytest tests -q -m "gpu and not slow" --timeout 120 -x -p no:cacheprovider > $OUT/tests.txt 2>&1; echo "rc=$?" >> $OUT/tests.txt
tail -3 $OUT/*.txt

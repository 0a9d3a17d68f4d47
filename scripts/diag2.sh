#!/bin/bash
OUT=gpurun_out/diag2; mkdir -p $OUT
export WGPF_DEBUG=1
timeout 120 python scripts/diag.py general > $OUT/general.txt 2>&1; echo "rc=$?" >> $OUT/general.txt
timeout 300 /usr/local/cuda/bin/compute-sanitizer --tool memcheck python scripts/diag.py general > $OUT/general_memcheck.txt 2>&1; echo "rc=$?" >> $OUT/general_memcheck.txt
timeout 120 python scripts/diag.py synth > $OUT/synth.txt 2>&1; echo "rc=$?" >> $OUT/synth.txt
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck python scripts/diag.py synth > $OUT/synth_memcheck.txt 2>&1; echo "rc=$?" >> $OUT/synth_memcheck.txt

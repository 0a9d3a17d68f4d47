#!/bin/bash
# ncu captures of the dominant kernels (one launch each, --set full, source
# counters): pass 1 (k_count_tps) and pass 2 (k_tps) of config 4, k_tpsd of
# config 5.  Usage (on the GPU box): bash scripts/prof_r02.sh <tag>
set -x
TAG=${1:-r02}
OUT=gpurun_out
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-p1"
ncu --set full --import-source on --clock-control none -k regex:k_count_tps -s 1 -c 1 \
    -o $OUT/${TAG}_count4 -f $B --no-config5 > $OUT/${TAG}_count4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_tps -s 1 -c 1 \
    -o $OUT/${TAG}_tps4 -f $B --no-config5 > $OUT/${TAG}_tps4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_tpsd -s 1 -c 1 \
    -o $OUT/${TAG}_tpsd5 -f $B --config 5 > $OUT/${TAG}_tpsd5.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $OUT/${TAG}_launches4.csv $B --no-config5 \
    > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $OUT/${TAG}_launches5.csv $B --config 5 \
    > /dev/null 2>&1
ls -la $OUT

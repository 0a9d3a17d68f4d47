bash scripts/ab_libs.sh ab_tps4 4 2
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-p1 --no-config5"
ncu --set full --import-source on --clock-control none -k k_tps -s 1 -c 1 \
    -o gpurun_out/r02b_tps4 -f $B > gpurun_out/r02b_tps4.log 2>&1
tail -3 gpurun_out/r02b_tps4.log

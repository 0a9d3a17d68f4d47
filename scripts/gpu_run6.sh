bash scripts/ab_libs.sh ab_deep5b 5 2
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-p1 --config 5"
ncu --set full --import-source on --clock-control none -k k_tpsd -s 1 -c 1 \
    -o gpurun_out/r02c_tpsd5 -f $B > gpurun_out/r02c_tpsd5.log 2>&1
tail -2 gpurun_out/r02c_tpsd5.log

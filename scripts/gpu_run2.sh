# A/B of the tail TMA map + source-level ncu captures of k_tps (config 4) and k_tpsd (config 5)
bash scripts/ab_env.sh ab_tail 4 "WGPF_NO_TAIL_MAP=1"
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-p1"
O=gpurun_out
ncu --set full --import-source on --clock-control none -k regex:'k_tps<' -s 1 -c 1 \
    -o $O/r02b_tps4 -f $B --no-config5 > $O/r02b_tps4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_tpsd -s 1 -c 1 \
    -o $O/r02b_tpsd5 -f $B --config 5 > $O/r02b_tpsd5.log 2>&1
ls -la $O

O=gpurun_out/g6; mkdir -p $O
for v in 0 256 128 0 256 128; do WGPF_TMA_L2=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-p1 --steps 10 > $O/l2_$v.json 2>/dev/null; python -c "
import json; d=json.load(open('$O/l2_$v.json')); print('$v', d['phases_ms']['emit'], d['phases_ms']['count'])" >> $O/ab.txt; done
KREGEX="^k_tps$" bash scripts/gpu_run.sh g6 ncu

# A/B: TMA record windows on / off (config 4, emit and count phases)
O=gpurun_out/${1:-tma}; mkdir -p $O
for v in on off on off; do
  if [ $v = off ]; then export WGPF_NO_TMA=1; else unset WGPF_NO_TMA; fi
  timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-p1 --steps 10 > $O/tma_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('$O/tma_$v.json')); print('$v', d['value']/1e9, d['phases_ms']['emit'], d['phases_ms']['count'])" >> $O/ab.txt
done

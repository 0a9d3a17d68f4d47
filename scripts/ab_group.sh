# A/B: k_tps lane mapping grouped by warp index (default) vs consecutive streams
O=gpurun_out/${1:-grp}; mkdir -p $O
for v in on off on off; do
  if [ $v = off ]; then export WGPF_NO_GROUP=1; else unset WGPF_NO_GROUP; fi
  timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-p1 --steps 10 > $O/grp_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('$O/grp_$v.json')); print('$v', d['value']/1e9, d['phases_ms']['emit'], d['phases_ms']['count'])" >> $O/ab.txt
done

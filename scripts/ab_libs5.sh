# A/B of alternative libwgpf builds on config 5 (k_tpsd)
O=gpurun_out/${1:-abl5}; mkdir -p $O
for rep in 1 2; do
for L in default paper_2505_21661_b200/_lib/ab/*.so; do
  if [ $L = default ]; then unset WGPF_LIB_OVERRIDE; else export WGPF_LIB_OVERRIDE=$PWD/$L; fi
  timeout 300 python bench.py --config 5 --no-e2e --no-cpu-baseline --no-p1 --steps 5 > $O/tmp.json 2>/dev/null
  python -c "
import json; d=json.load(open('$O/tmp.json')); print('$(basename $L)', d['value']/1e9, d['phases_ms']['emit'])" >> $O/ab.txt
done; done

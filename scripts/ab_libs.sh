# A/B of alternative builds of libwgpf (paper_2505_21661_b200/_lib/ab/*.so) vs the default
O=gpurun_out/${1:-abl}; mkdir -p $O
for rep in 1 2; do
for L in default paper_2505_21661_b200/_lib/ab/*.so; do
  if [ $L = default ]; then unset WGPF_LIB_OVERRIDE; else export WGPF_LIB_OVERRIDE=$PWD/$L; fi
  timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-p1 --steps 10 > $O/tmp.json 2>/dev/null
  python -c "
import json; d=json.load(open('$O/tmp.json')); print('$(basename $L)', d['value']/1e9, d['phases_ms']['emit'], d['phases_ms']['count'])" >> $O/ab.txt
done; done

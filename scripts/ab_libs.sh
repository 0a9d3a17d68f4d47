# A/B of alternative builds of libwgpf (paper_2505_21661_b200/_lib/ab/*.so) vs the default
# usage: bash scripts/ab_libs.sh <tag> [config (4|5)] [reps]
O=gpurun_out/${1:-abl}; CFG=${2:-4}; REPS=${3:-2}; mkdir -p $O
X="--no-config5"; [ "$CFG" = 5 ] && X=""
for rep in $(seq $REPS); do
for L in default paper_2505_21661_b200/_lib/ab/*.so; do
  if [ $L = default ]; then unset WGPF_LIB_OVERRIDE; else export WGPF_LIB_OVERRIDE=$PWD/$L; fi
  timeout 300 python bench.py --config $CFG $X --no-e2e --no-cpu-baseline --no-p1 --steps 10 > $O/tmp.json 2>$O/tmp.err
  python -c "
import json; d=json.load(open('$O/tmp.json')); p=d['phases_ms']
print('%-16s %7.2f G/s step %.3f count %.3f emit %.3f' % ('$(basename $L)', d['value']/1e9, d['ms_per_step'], p['count'], p['emit']))" >> $O/ab.txt 2>&1 || tail -3 $O/tmp.err >> $O/ab.txt
done; done
cat $O/ab.txt

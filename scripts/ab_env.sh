# A/B of run-time switches: bash scripts/ab_env.sh <tag> <config> "<ENV=1 ...>" ["<ENV2=1>" ...]
# Alternates the default with each variant (3 rounds); prints G records/s, step ms and
# the count / emit phases of bench.py (headline config only).
O=gpurun_out/${1:-abe}; CFG=${2:-4}; shift 2; mkdir -p $O
for rep in 1 2 3; do
for V in "default" "$@"; do
  if [ "$V" = default ]; then E=""; else E="$V"; fi
  env $E timeout 300 python bench.py --config $CFG --no-e2e --no-cpu-baseline --no-p1 --no-config5 --steps 10 > $O/tmp.json 2>$O/tmp.err
  python -c "
import json; d=json.load(open('$O/tmp.json')); p=d['phases_ms']
print('%-28s %7.2f G/s step %.3f count %.3f emit %.3f' % ('$V', d['value']/1e9, d['ms_per_step'], p['count'], p['emit']))" >> $O/ab.txt 2>&1 || tail -3 $O/tmp.err >> $O/ab.txt
done; done
cat $O/ab.txt

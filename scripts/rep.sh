# repeated config-4 bench runs (emit / count phases), env from the caller
O=gpurun_out/${1:-rep}; N=${2:-4}; mkdir -p $O
for i in $(seq $N); do
  timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-p1 --steps 10 > $O/r$i.json 2>/dev/null
  python -c "
import json; d=json.load(open('$O/r$i.json')); print('$i', d['value']/1e9, d['phases_ms']['emit'], d['phases_ms']['count'], d['ms_per_step'])" >> $O/rep.txt
done

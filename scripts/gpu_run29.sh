timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest29.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gputest29.log
for rep in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline --no-p1 --no-config5 --e2e-steps 4 --steps 3 --warmup 3 --shim-streams 0 > gpurun_out/b29.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/b29.json')); e=d['e2e']
print('trim', round(e['value']/1e9,3), 'ms', round(e['ms_per_step'],1), 'pageable', round(e['pageable']['value']/1e9,3), round(e['pageable']['ms_per_step'],1))"
done

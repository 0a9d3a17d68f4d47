timeout 900 python -m pytest tests -m gpu -x -q -k "pipelin or image or shim or cli" > gpurun_out/gputest31.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gputest31.log
for rep in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline --no-p1 --no-config5 --e2e-steps 4 --steps 3 --warmup 3 > gpurun_out/b31.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/b31.json')); e=d['e2e']
print('e2e', round(e['value']/1e9,3), 'ms', round(e['ms_per_step'],1), 'pageable', round(e['pageable']['value']/1e9,3), 'shim', d['e2e_shim']['value']/1e6)"
done

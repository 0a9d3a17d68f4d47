timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest7.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/gputest7.log
for c in 5 4; do for r in 1 2; do
timeout 300 python bench.py --config $c --no-config5 --no-e2e --no-cpu-baseline --no-p1 --steps 10 > gpurun_out/b7_$c.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/b7_$c.json')); p=d['phases_ms']
print('config $c %7.2f G/s step %.3f count %.3f emit %.3f frac_step %.3f' % (d['value']/1e9, d['ms_per_step'], p['count'], p['emit'], d['hbm_frac_step']))"
done; done

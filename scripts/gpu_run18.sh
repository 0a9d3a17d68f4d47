timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest18.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/gputest18.log
timeout 900 python bench.py > gpurun_out/bench18.log 2> gpurun_out/bench18.err; echo "bench rc=$?"
python - <<'PY'
import json
d=[json.loads(l) for l in open('gpurun_out/bench18.log') if l.startswith('{')][-1]
print({k:d[k] for k in ['value','ms_per_step','hbm_frac_step']}, d['phases_ms'], d['roofline']['frac'])
print('p1', {k:d['p1'][k] for k in ['value','t_plain_ms','t_instr_ms','accuracy_rel_err','record_cost_cycles','flush_cycles_per_cta']})
c=d['config5']; print('c5', c['ms_per_step'], c['hbm_frac_step'], c['roofline']['frac'], c['phases_ms'])
print('e2e', d['e2e']['value'], d['e2e']['pageable']['value'], 'shim', d['e2e_shim'])
print('cpu', d['cpu_baseline']['value'], d['clocks'])
PY
python -c "import __graft_entry__ as g; g.smoke()"

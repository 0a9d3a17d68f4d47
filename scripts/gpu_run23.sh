timeout 1800 python scripts/fuzz_sweep.py 25 > gpurun_out/fuzz_sweep.log 2>&1; echo "fuzz rc=$?"; tail -8 gpurun_out/fuzz_sweep.log
timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-p1 --no-config5 --steps 10 > gpurun_out/b23.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b23.json')); print(d['stats_only'], d['roofline'])"

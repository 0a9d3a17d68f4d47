for rep in 1 2; do for MB in 256 128 512 1024; do
  WGPF_CHUNK_MB=$MB timeout 600 python bench.py --no-cpu-baseline --no-p1 --no-config5 --e2e-steps 4 --steps 3 --warmup 3 --shim-streams 0 > gpurun_out/b30.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/b30.json')); e=d['e2e']
print('chunk $MB', round(e['value']/1e9,3), 'ms', round(e['ms_per_step'],1), 'pageable', round(e['pageable']['value']/1e9,3))"
done; done

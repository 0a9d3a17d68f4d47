for rep in 1 2; do for L in default trim; do
  if [ $L = default ]; then unset WGPF_LIB_OVERRIDE; else export WGPF_LIB_OVERRIDE=$PWD/paper_2505_21661_b200/_lib/ab/$L.so; fi
  timeout 600 python bench.py --no-cpu-baseline --no-p1 --no-config5 --e2e-steps 4 --steps 3 --warmup 3 --shim-streams 0 > gpurun_out/b28.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/b28.json')); e=d['e2e']
print('$L', round(e['value']/1e9,3), 'ms', round(e['ms_per_step'],1), 'pageable', round(e['pageable']['value']/1e9,3))"
done; done
unset WGPF_LIB_OVERRIDE
WGPF_LIB_OVERRIDE=$PWD/paper_2505_21661_b200/_lib/ab/trim.so timeout 900 python -m pytest tests -m gpu -x -q -k "pipelin or image or chunk or shim or cli or multi" > gpurun_out/gputest28.log 2>&1; echo "trim tests rc=$?"; tail -2 gpurun_out/gputest28.log

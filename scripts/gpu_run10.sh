timeout 600 python -m pytest tests -m gpu -x -q -k "p1 or gemm or align or attn" > gpurun_out/gputest10.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest10.log
for m in 1 2 1 2; do WGPF_P1_MODE=$m timeout 300 python bench_p1.py | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('mode $m', {k:d[k] for k in d if k in ('overhead_pct','t_plain_ms','t_instr_ms','accuracy_rel_err')})"; done

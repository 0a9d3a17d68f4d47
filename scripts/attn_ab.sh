# A/B of compile-time attention variants (paper_2505_21661_b200/_lib/ab_p1/*.so):
#   bash scripts/attn_ab.sh "v1 v2 ..." [reps]   (config 3, B=16 H=16 S=8192)
python -c "from paper_2505_21661_b200 import _build as b; b.build_p1(); b.build()" || exit 1
for rep in $(seq ${2:-1}); do for v in $1; do
  echo -n "$v "; WGPF_P1_LIB_OVERRIDE=paper_2505_21661_b200/_lib/ab_p1/$v.so timeout 300 python -c "
import sys, json; sys.path.insert(0,'.')
import bench_p1
r = bench_p1.measure_attn(iters=10, warmup=3, analyse=False)
d, s = r['kv_double_buffered'], r['kv_single_buffered_fa3_vanilla']
print(json.dumps({'kv1': [round(s['tflops_plain']), round(s['overhead_pct'], 2)], 'kv2': [round(d['tflops_plain']), round(d['overhead_pct'], 2)], 'sdpa': round(r['sdpa_tflops'])}))
" 2>&1 | tail -1
done; done

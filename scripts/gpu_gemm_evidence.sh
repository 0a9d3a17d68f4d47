# P1 GEMM evidence (profiles/r02_gemm_pair*): GPU tests of the P1 path,
# bench_p1, pair / single-CTA A/B, ncu launch list and one --set full capture.
#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2505_21661_b200 import _build as b; b.build_p1(); b.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_p1.py tests/test_gpu_align.py tests/test_gpu_p1_runtime.py -q -x > gpurun_out/gputest45.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest45.log
timeout 600 python bench_p1.py > gpurun_out/r02_gemm_pair.json 2> gpurun_out/bench_p1.err; echo "bench_p1 rc=$?"
python - <<'PY'
import json
d=json.load(open("gpurun_out/r02_gemm_pair.json"))
print({k: d[k] for k in ("value","t_plain_ms","t_instr_ms","tflops_plain","tflops_instr","tflops_cublas","accuracy_rel_err","smem_total_bytes_per_cta","sass_instructions","instrumented_output_identical","scope_means_cycles")})
PY
for i in 1 2 3; do timeout 120 python scripts/gemm_pair_check.py time 2>&1 | tail -1; done > gpurun_out/r02_gemm_pair_ab.log
WGPF_GEMM_SINGLE=1 timeout 120 python scripts/gemm_pair_check.py time 2>&1 | tail -1 >> gpurun_out/r02_gemm_pair_ab.log
cat gpurun_out/r02_gemm_pair_ab.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_gemm --csv --log-file gpurun_out/r02_gemm_launches.csv python scripts/gemm_pair_check.py time > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 2 -c 2 -o gpurun_out/r02_gemm_pair -f python scripts/gemm_pair_check.py time > gpurun_out/ncu_gemm.log 2>&1; echo "ncu2 rc=$?"

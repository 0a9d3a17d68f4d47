timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest13.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/gputest13.log
tests/cxx/_build/shim_bench 524288 2
python scripts/time_k6.py 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('wide', d['k_fast_emit'])"
WGPF_NO_WIDE=1 python scripts/time_k6.py 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('warp', d['k_fast_emit'])"

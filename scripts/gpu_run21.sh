bash scripts/ab_libs.sh ab21 5 2
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "deep or wide or full_config5 or 64k" > gpurun_out/gputest21.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest21.log

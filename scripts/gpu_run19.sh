timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_p1.py -m gpu -x -q > gpurun_out/gputest19.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/gputest19.log
tests/cxx/_build/shim_bench 524288 2

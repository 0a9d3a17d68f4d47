timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest12.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest12.log
tests/cxx/_build/shim_bench 524288 2

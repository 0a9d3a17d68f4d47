timeout 900 python -m pytest tests -m gpu -x -q -k "shim or cli or decode or image" > gpurun_out/gputest32.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gputest32.log
tests/cxx/_build/shim_bench 524288 2

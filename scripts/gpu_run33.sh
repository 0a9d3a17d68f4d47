timeout 900 python -m pytest tests -m gpu -x -q -k "mean or fixture or shim or stats" > gpurun_out/gputest33.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gputest33.log
tests/cxx/_build/shim_bench 524288 2

timeout 1200 python -m pytest tests -m gpu -x -q -k "shim or cli or stats or mean or chrome or critical or report" > gpurun_out/gputest20.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/gputest20.log
tests/cxx/_build/shim_bench 524288 2

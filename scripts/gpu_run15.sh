timeout 1200 python -m pytest tests -m gpu -x -q -k "mean or fixture or shim or cli or report or oracle or stats" > gpurun_out/gputest15.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest15.log
tests/cxx/_build/shim_bench 524288 2

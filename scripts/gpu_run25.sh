bash scripts/ab_libs.sh ab25 4 2
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest25.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest25.log

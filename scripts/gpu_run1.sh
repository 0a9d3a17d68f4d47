set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
cat MEASURED_PEAKS.json 2>/dev/null
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/gputest.log
timeout 600 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 6000 gpurun_out/bench.log

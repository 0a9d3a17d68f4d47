# Round-end validation on one GPU box: the GPU tests, smoke(), the default
# bench line and the reference arm (outputs under gpurun_out/validate/).
#   /usr/local/graft/bin/gpurun --timeout 2700 -- bash scripts/gpu_validate.sh
O=gpurun_out/validate; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/ref_arm.json 2> $O/ref_arm.err; echo "ref rc=$?"

timeout 1200 python -m pytest tests -m gpu -x -q -k "p1 or gemm or flush or align or attn" > gpurun_out/gputest16.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest16.log
python -c "import bench_p1, json; print(json.dumps(bench_p1.measure_flush()))"
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-p1"
ncu --set full --import-source on --clock-control none -k regex:k_count_tps -s 1 -c 1 \
    -o gpurun_out/r02_count5 -f $B --config 5 > gpurun_out/r02_count5.log 2>&1; tail -1 gpurun_out/r02_count5.log

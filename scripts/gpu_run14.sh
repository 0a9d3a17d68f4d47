ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/shim_launches.csv tests/cxx/_build/shim_bench 524288 1 > gpurun_out/shim_ncu.out 2>&1
python scripts/time_k6.py > gpurun_out/r02_k6_wide.json 2> gpurun_out/time_k6.err; cat gpurun_out/r02_k6_wide.json

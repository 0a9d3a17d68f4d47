# Round-2 final (after the exact-pitch deep windows): tests, smoke, seed sweep,
# bench line, ncu of k_tpsd + launch list of config 5, sanitizers
O=gpurun_out/final3; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 1800 python scripts/fuzz_sweep.py 25 > $O/fuzz_sweep.log 2>&1; echo "fuzz rc=$?"; tail -2 $O/fuzz_sweep.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-p1"
ncu --set full --import-source on --clock-control none -k regex:k_tpsd -s 1 -c 1 \
    -o $O/r02_tpsd5 -f $B --config 5 > $O/r02_tpsd5.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $O/r02_launches_config5.csv $B --config 5 > /dev/null 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/san_driver.py \
    > $O/r02_sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?" >> $O/r02_sanitizer_$tool.txt
  tail -2 $O/r02_sanitizer_$tool.txt
done
python scripts/time_k6.py > $O/r02_k6_wide.json 2>/dev/null

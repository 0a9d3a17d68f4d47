# Round-2 evidence with the final kernels: ncu captures of the dominant kernels,
# launch lists, the reference arm, sanitizer logs.  Output under gpurun_out/ev/.
O=gpurun_out/ev; mkdir -p $O
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-p1"
ncu --set full --import-source on --clock-control none -k k_tps -s 1 -c 1 \
    -o $O/r02_tps4 -f $B --no-config5 > $O/r02_tps4.log 2>&1; tail -1 $O/r02_tps4.log
ncu --set full --import-source on --clock-control none -k k_tpsd -s 1 -c 1 \
    -o $O/r02_tpsd5 -f $B --config 5 > $O/r02_tpsd5.log 2>&1; tail -1 $O/r02_tpsd5.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $O/r02_launches_config4.csv $B --no-config5 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $O/r02_launches_config5.csv $B --config 5 > /dev/null 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/ref_arm.json 2> $O/ref_arm.err; echo "ref rc=$?"; tail -c 1500 $O/ref_arm.json
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/san_driver.py \
    > $O/r02_sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?" >> $O/r02_sanitizer_$tool.txt
  tail -3 $O/r02_sanitizer_$tool.txt
done
ls -la $O

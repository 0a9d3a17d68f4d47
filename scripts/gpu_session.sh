#!/bin/bash
# One GPU session: tests, bench, ncu launch list + full capture of the decode
# kernel.  Usage (under gpurun): bash scripts/gpu_session.sh [tag] [what...]
# what: tests p1 bench ncu benchall   (default: tests bench ncu)
set -u
TAG=${1:-s}; shift || true
WHAT=${*:-"tests bench ncu"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
nproc > $OUT/nproc.txt; lscpu | head -20 >> $OUT/nproc.txt
for w in $WHAT; do
case $w in
tests)
  timeout 1200 python -m pytest tests -x -q -m "gpu and not slow" > $OUT/tests.txt 2>&1; echo "tests rc=$?" >> $OUT/tests.txt ;;
testsall)
  timeout 1800 python -m pytest tests -q -m gpu > $OUT/tests_all.txt 2>&1; echo "rc=$?" >> $OUT/tests_all.txt ;;
p1)
  timeout 900 python -m pytest tests/test_gpu_p1.py -x -q > $OUT/p1.txt 2>&1; echo "rc=$?" >> $OUT/p1.txt ;;
smoke)
  timeout 600 python __graft_entry__.py smoke > $OUT/smoke.txt 2>&1; echo "rc=$?" >> $OUT/smoke.txt ;;
benchsmall)
  timeout 600 python bench.py --streams 262144 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_small.json 2> $OUT/bench_small.err ;;
bench)
  timeout 1500 python bench.py > $OUT/bench.json 2> $OUT/bench.err ;;
benchref)
  timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err ;;
ncu)
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_bench.log 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_fast_emit -s 1 -c 1 \
    -o $OUT/emit python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_full.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_count_fast -s 1 -c 1 \
    -o $OUT/count python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_count.log 2>&1 ;;
esac
done
ls -la $OUT

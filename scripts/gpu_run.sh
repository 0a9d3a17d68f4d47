#!/bin/bash
# usage: bash scripts/gpu_run.sh TAG "steps..."   steps: smoke tests p1 overlap benchsmall bench benchref ncu
TAG=$1; shift; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
for st in $*; do case $st in
smoke) timeout 300 python __graft_entry__.py smoke > $OUT/smoke.txt 2>&1; echo "rc=$?" >> $OUT/smoke.txt ;;
tests) timeout 1200 python -m pytest tests -q -m "gpu and not slow" --timeout 300 -p no:cacheprovider -k "not test_gpu_p1 and not test_gpu_overlap" > $OUT/tests.txt 2>&1; echo "rc=$?" >> $OUT/tests.txt ;;
p1) timeout 600 python -m pytest tests/test_gpu_p1.py -q --timeout 200 -p no:cacheprovider > $OUT/p1.txt 2>&1; echo "rc=$?" >> $OUT/p1.txt ;;
overlap) timeout 600 python -m pytest tests/test_gpu_overlap.py -q --timeout 200 -p no:cacheprovider > $OUT/overlap.txt 2>&1; echo "rc=$?" >> $OUT/overlap.txt ;;
slow) timeout 900 python -m pytest tests -q -m "slow" --timeout 800 -p no:cacheprovider > $OUT/slow.txt 2>&1; echo "rc=$?" >> $OUT/slow.txt ;;
benchsmall) timeout 400 python bench.py --streams 262144 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_small.json 2> $OUT/bench_small.err ;;

parity) timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 300 -p no:cacheprovider > $OUT/parity.txt 2>&1; echo "rc=$?" >> $OUT/parity.txt ;;
quick) timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-p1 > $OUT/quick.json 2> $OUT/quick.err ;;
bench) timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err ;;
bench5) timeout 1200 python bench.py --config 5 --no-p1 > $OUT/bench5.json 2> $OUT/bench5.err ;;
benchref) timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err ;;
benchp1) timeout 600 python bench_p1.py > $OUT/bench_p1.json 2> $OUT/bench_p1.err ;;
ncu) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_bench.log 2>&1
     timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-^k_tps$} -s 1 -c 1 -o $OUT/emit python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_full.log 2>&1 ;;
ncusmall) timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_small.csv python bench.py --streams 262144 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_bench_small.log 2>&1
     timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_tps} -s 1 -c 1 -o $OUT/emit_small python bench.py --streams 262144 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_full_small.log 2>&1 ;;
split) for fl in 0 8 1 9; do WGPF_BENCH_FLAGS=$fl timeout 400 python bench.py --streams 1048576 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-p1 > $OUT/split_$fl.json 2>> $OUT/split.err; done ;;
p1ab) for m in 1 2 1 2; do WGPF_P1_MODE=$m timeout 300 python bench_p1.py > $OUT/p1_mode$m.json 2>> $OUT/p1ab.err; cat $OUT/p1_mode$m.json >> $OUT/p1ab.jsonl; done ;;
merge) timeout 300 python -m pytest tests/test_gpu_parity.py -q -k merge -p no:cacheprovider -vv > $OUT/merge.txt 2>&1 ;;
esac; done

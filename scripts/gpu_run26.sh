bash scripts/ab_libs.sh ab26 5 2
for L in p32w13 p32w12; do
WGPF_LIB_OVERRIDE=$PWD/paper_2505_21661_b200/_lib/ab/$L.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "deep or wide or 64k or config5" > gpurun_out/gputest26_$L.log 2>&1; echo "$L parity rc=$?"; tail -2 gpurun_out/gputest26_$L.log
done

bash scripts/ab_libs.sh ab17_c4 4 2
bash scripts/ab_libs.sh ab17_c5 5 1
WGPF_LIB_OVERRIDE=$PWD/paper_2505_21661_b200/_lib/ab/wstat.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "not full" > gpurun_out/gputest17.log 2>&1; echo "wstat parity rc=$?"; tail -3 gpurun_out/gputest17.log

bash scripts/ab_libs.sh ab27c4 4 2
bash scripts/ab_libs.sh ab27c5 5 1
WGPF_LIB_OVERRIDE=$PWD/paper_2505_21661_b200/_lib/ab/b3.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "not full" > gpurun_out/gputest27.log 2>&1; echo "b3 parity rc=$?"; tail -2 gpurun_out/gputest27.log

bash scripts/ab_libs.sh ab22 5 2
WGPF_LIB_OVERRIDE=$PWD/paper_2505_21661_b200/_lib/ab/cntg13.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "deep or wide or 64k" > gpurun_out/gputest22.log 2>&1; echo "cntg13 parity rc=$?"; tail -3 gpurun_out/gputest22.log

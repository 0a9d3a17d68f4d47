bash scripts/ab_libs.sh ab24c5 5 2
bash scripts/ab_libs.sh ab24c4 4 1
WGPF_LIB_OVERRIDE=$PWD/paper_2505_21661_b200/_lib/ab/tmae5.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "deep or wide or 64k or fuzz or config5" > gpurun_out/gputest24.log 2>&1; echo "tmae5 parity rc=$?"; tail -3 gpurun_out/gputest24.log

timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "full_config5 or full_size_fast" > gpurun_out/gputest11.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/gputest11.log
bash scripts/ab_env.sh ab_l2 4 "WGPF_TMA_L2=128" "WGPF_TMA_L2=64" "WGPF_TMA_L2=0"
bash scripts/ab_libs.sh ab_shfl 4 2

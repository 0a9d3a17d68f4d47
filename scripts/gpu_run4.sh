# overlapped pass 1 / pass 2: parity tests, then A/B (overlap off / default / co1)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest4.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/gputest4.log
bash scripts/ab_env.sh ab_ovl 4 "WGPF_NO_OVERLAP=1"
bash scripts/ab_libs.sh ab_ovl_libs 4 1

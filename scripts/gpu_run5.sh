# k_tpsd: marker-free specialisation, first-key shortcut, on-demand cp.async slots; A/B on config 5
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest5.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/gputest5.log
bash scripts/ab_libs.sh ab_deep5 5 2

# scratch GPU job (edited per experiment)
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python -m pytest tests -m gpu -q -x --timeout=120 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
TV_CONFIGS=configs2,configs4,configs3 TV_MODES=s1p0 timeout 400 python tools/time_variants.py 2>&1 | tee gpurun_out/tv.log
TV_CONFIGS=configs2 TV_MODES=s1p0 timeout 400 python tools/time_variants.py 2>&1 | tee -a gpurun_out/tv.log

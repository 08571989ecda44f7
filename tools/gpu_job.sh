# scratch GPU job (edited per experiment)
timeout 600 python -m pytest tests -m gpu -q -x --timeout=120 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
TV_CONFIGS=configs1 TV_MODES=s1p0 timeout 400 python tools/time_variants.py 2>&1 | tee gpurun_out/tv.log

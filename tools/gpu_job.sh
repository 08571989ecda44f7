# scratch GPU job (edited per experiment)
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
TV_CONFIGS=configs2,configs4,configs3,configs0,configs1 TV_MODES=s1p0 timeout 900 python tools/time_variants.py 2>&1 | tee gpurun_out/tv.log

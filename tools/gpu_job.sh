# scratch GPU job (edited per experiment)
timeout 300 python tools/trace_step.py configs2 2>&1 | tee gpurun_out/trace.log | head -8
mv tools/_variants/trace.so /tmp/
TV_CONFIGS=configs2,configs4,configs3,configs0 TV_MODES=s1p0 timeout 300 python tools/time_variants.py 2>&1 | tee gpurun_out/tv.log
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log

# scratch GPU job (edited per experiment)
timeout 900 python -m pytest tests -m gpu -q -x --timeout=120 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline --no-other-configs > gpurun_out/bench.log 2>&1; echo "bench rc=$?"

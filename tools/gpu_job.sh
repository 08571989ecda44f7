# scratch GPU job (edited per experiment)
timeout 300 python tools/trace_step.py configs2 2>&1 | tee gpurun_out/trace.log | head -8

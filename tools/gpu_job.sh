# scratch GPU job (edited per experiment)
TV_CONFIGS=configs2 TV_MODES=s1p0 timeout 300 python tools/time_variants.py 2>&1 | tee gpurun_out/tv.log

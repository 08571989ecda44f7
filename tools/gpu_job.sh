# scratch GPU job (edited per experiment)
TV_CONFIGS=configs1 TV_MODES=s1p0 timeout 400 python tools/time_variants.py 2>&1 | tee gpurun_out/tv.log
TV_CONFIGS=configs1 TV_MODES=s1p0 timeout 400 python tools/time_variants.py 2>&1 | tee -a gpurun_out/tv.log

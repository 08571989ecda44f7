# Round measurement on one B200 (run through gpurun): GPU tests, smoke,
# bench (+ reference arm), launch list and a full ncu capture of one step
# (configs[2]); summaries go to profiles/ by hand (tools/ncu_summary.py,
# tools/ncu_stalls.py, tools/ncu_mix.py).
timeout 900 python -m pytest tests -m gpu -q --timeout=120 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "bench ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage -s 3 -c 3 -o /tmp/step_full python tools/profile_step.py --schedule 1 --steps 2 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py /tmp/step_full.ncu-rep gpurun_out/ncu_step 1048576 > /dev/null 2>&1
(for i in 0 1 2; do python tools/ncu_stalls.py /tmp/step_full.ncu-rep $i; python tools/ncu_mix.py /tmp/step_full.ncu-rep $i | tail -2; done) > gpurun_out/ncu_stalls.txt 2>&1

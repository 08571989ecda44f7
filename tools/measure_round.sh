# Round measurement on one B200 (run through gpurun): GPU tests, smoke,
# bench (+ reference arm), launch list, full ncu captures of one configs[2]
# step, the configs[0] resident kernel and the configs[1] 3-flavour stages.
# Summaries go to profiles/ by hand (tools/ncu_summary.py, tools/ncu_stalls.py,
# tools/ncu_mix.py).  usage: bash tools/measure_round.sh [tag]
TAG=${1:-r12}
timeout 1500 python -m pytest tests -m gpu -q --timeout=600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_short.log 2>&1; echo "bench short rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "bench ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage -s 3 -c 3 -o /tmp/${TAG}_step python tools/profile_step.py --schedule 1 --steps 2 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_resident -c 1 -o /tmp/${TAG}_resident0 env N=50 python tools/profile_resident.py > gpurun_out/ncu_res.log 2>&1; echo "ncu resident rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage3 -s 3 -c 3 -o /tmp/${TAG}_flav3 python tools/profile_step.py --config configs1 --schedule 1 --steps 2 > gpurun_out/ncu_flav3.log 2>&1; echo "ncu flav3 rc=$?"
# summaries (the reports stay on the box: gpurun copies back at most 64 MiB)
python tools/ncu_summary.py /tmp/${TAG}_step.ncu-rep gpurun_out/${TAG}_ncu_step 1048576 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/${TAG}_resident0.ncu-rep gpurun_out/${TAG}_ncu_resident0 25600 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/${TAG}_flav3.ncu-rep gpurun_out/${TAG}_ncu_flav3 65536 > /dev/null 2>&1
(for i in 0 1 2; do python tools/ncu_stalls.py /tmp/${TAG}_step.ncu-rep $i; python tools/ncu_mix.py /tmp/${TAG}_step.ncu-rep $i | tail -2; done) > gpurun_out/${TAG}_ncu_stalls.txt 2>&1
(python tools/ncu_stalls.py /tmp/${TAG}_resident0.ncu-rep 0; python tools/ncu_mix.py /tmp/${TAG}_resident0.ncu-rep 0 | tail -2) > gpurun_out/${TAG}_ncu_resident0_stalls.txt 2>&1
(for i in 0 1 2; do python tools/ncu_stalls.py /tmp/${TAG}_flav3.ncu-rep $i; python tools/ncu_mix.py /tmp/${TAG}_flav3.ncu-rep $i | tail -2; done) > gpurun_out/${TAG}_ncu_flav3_stalls.txt 2>&1
ncu -i /tmp/${TAG}_step.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/${TAG}_step_dram.csv 2>&1
ls -la gpurun_out

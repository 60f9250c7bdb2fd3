cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/r3y_smi.txt
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/r3y_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r3y_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3y_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r3y_smoke.log
timeout 1800 python bench.py > gpurun_out/r3y_bench.json 2> gpurun_out/r3y_bench.err; echo "bench rc=$?" >> gpurun_out/r3y_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r3y_ref.json 2> gpurun_out/r3y_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r3y_launches.csv python bench.py --steps 2 --warmup 3 --no-si --no-e2e --no-solve --no-kernels --no-cpu --no-generic > gpurun_out/r3y_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -f -o gpurun_out/r3y_sweep_c5 python tools/sweep_c5_once.py 3 > gpurun_out/r3y_ncu_sweep.log 2>&1
ncu -i gpurun_out/r3y_sweep_c5.ncu-rep --page details > gpurun_out/r3y_sweep_c5_details.txt 2>/dev/null
ncu -i gpurun_out/r3y_sweep_c5.ncu-rep --page raw --csv > gpurun_out/r3y_sweep_c5_raw.csv 2>/dev/null
rm -f gpurun_out/r3y_sweep_c5.ncu-rep
tail -3 gpurun_out/r3y_tests.log; tail -2 gpurun_out/r3y_smoke.log; head -c 400 gpurun_out/r3y_bench.json
timeout 600 python bench.py --steps 40 --no-si --no-e2e --no-solve --no-kernels --no-cpu --no-generic > gpurun_out/r3y_bench40.json 2>> gpurun_out/r3y_bench.err
timeout 900 python tools/shard_probe.py 1 2 4 8 > gpurun_out/r3y_shard.jsonl 2>> gpurun_out/r3y_bench.err

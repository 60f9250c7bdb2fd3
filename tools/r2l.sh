cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/r2l_smi.txt
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2l_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2l_tests.log
timeout 1200 python bench.py > gpurun_out/r2l_bench.json 2> gpurun_out/r2l_bench.err; echo "bench rc=$?" >> gpurun_out/r2l_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2l_ref.json 2> gpurun_out/r2l_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2l_launches.csv python bench.py --steps 2 --warmup 3 --no-si --no-e2e --no-solve --no-kernels --no-cpu --no-generic > gpurun_out/r2l_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o gpurun_out/r2l_sweep_c5 python tools/sweep_c5_once.py 3 > gpurun_out/r2l_ncu_sweep.log 2>&1
ncu -i gpurun_out/r2l_sweep_c5.ncu-rep --page details > gpurun_out/r2l_sweep_c5_details.txt 2>/dev/null
ncu -i gpurun_out/r2l_sweep_c5.ncu-rep --page raw --csv > gpurun_out/r2l_sweep_c5_raw.csv 2>/dev/null
rm -f gpurun_out/r2l_sweep_c5.ncu-rep
GN=24 timeout 900 ncu --set full --clock-control none -k regex:"apply_L_block|sweep_block|d2m_kernel|m2d_kernel|coarse_gs_kernel" -c 6 -o gpurun_out/r2l_generic python tools/generic_probe.py > gpurun_out/r2l_ncu_generic.log 2>&1
ncu -i gpurun_out/r2l_generic.ncu-rep --page details > gpurun_out/r2l_generic_details.txt 2>/dev/null
rm -f gpurun_out/r2l_generic.ncu-rep
for n in 64 128 256; do timeout 300 python tools/gs_probe.py 4 10 $n >> gpurun_out/r2l_gs_c4_sizes.log 2>&1; done
timeout 900 python bench.py --steps 3 --no-si --no-e2e --no-cpu --no-kernels --no-generic --solve-configs 4 > gpurun_out/r2l_bench_c4.json 2> gpurun_out/r2l_bench_c4.err

cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r3e_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r3e_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3e_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r3e_smoke.log
timeout 1500 python bench.py > gpurun_out/r3e_bench.json 2> gpurun_out/r3e_bench.err; echo "bench rc=$?" >> gpurun_out/r3e_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r3e_ref.json 2> gpurun_out/r3e_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r3e_launches.csv python bench.py --steps 2 --warmup 3 --no-si --no-e2e --no-solve --no-kernels --no-cpu --no-generic > gpurun_out/r3e_ncu_launch.log 2>&1
for k in apply_L_mma sweep_mma d2m_block m2d_block coarse_gs_flow; do
  GN=24 timeout 600 ncu --set full --clock-control none -k regex:$k -s 1 -c 1 -o gpurun_out/r3e_$k python tools/generic_probe.py > gpurun_out/r3e_ncu_$k.log 2>&1
  ncu -i gpurun_out/r3e_$k.ncu-rep --page details > gpurun_out/r3e_${k}_details.txt 2>/dev/null
  rm -f gpurun_out/r3e_$k.ncu-rep
done
GN=24 timeout 300 python tools/generic_probe.py > gpurun_out/r3e_gen24.json 2>&1

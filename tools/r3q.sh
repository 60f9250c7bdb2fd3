cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/r3q_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r3q_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3q_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r3q_smoke.log
timeout 1800 python bench.py > gpurun_out/r3q_bench.json 2> gpurun_out/r3q_bench.err; echo "bench rc=$?" >> gpurun_out/r3q_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r3q_ref.json 2> gpurun_out/r3q_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r3q_launches.csv python bench.py --steps 2 --warmup 3 --no-si --no-e2e --no-solve --no-kernels --no-cpu --no-generic > gpurun_out/r3q_ncu_launch.log 2>&1
tail -3 gpurun_out/r3q_tests.log; cat gpurun_out/r3q_smoke.log | tail -2; head -c 600 gpurun_out/r3q_bench.json

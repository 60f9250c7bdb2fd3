cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/r2u_smi.txt
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2u_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2u_tests.log
timeout 1200 python bench.py > gpurun_out/r2u_bench.json 2> gpurun_out/r2u_bench.err; echo "bench rc=$?" >> gpurun_out/r2u_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2u_ref.json 2> gpurun_out/r2u_ref.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2u_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2u_smoke.log

cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt
timeout 900 python -m pytest tests/test_gpu_sharded_emulation.py tests/test_gpu_fold_gate.py tests/test_gpu_c4n64_golden.py -m gpu -q -k "not test_solve" > gpurun_out/r2a_new.log 2>&1; echo "new rc=$?" >> gpurun_out/r2a_new.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2a_all.log 2>&1; echo "all rc=$?" >> gpurun_out/r2a_all.log

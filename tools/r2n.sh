cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for i in 1 2; do
for v in default nst4 nst8 nst10; do
  if [ $v = default ]; then timeout 300 python tools/sweep_ab.py 10 >> gpurun_out/r2n_nst.log 2>&1
  else STAMG_LIB=abl/$v.so timeout 300 python tools/sweep_ab.py 10 >> gpurun_out/r2n_nst.log 2>&1; fi
done; done
timeout 900 python -m pytest tests/test_gpu_krylov_workspace.py tests/test_gpu_shard_sweep.py tests/test_gpu_coarse_cluster.py -m gpu -q > gpurun_out/r2n_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2n_tests.log

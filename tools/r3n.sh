cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_shard_sweep.py -m gpu -q -x > gpurun_out/r3n_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3n_tests.log
tail -3 gpurun_out/r3n_tests.log
for v in default m2d_ef sweep_old default; do
  echo "== $v" >> gpurun_out/r3n_ab.log
  if [ "$v" = default ]; then timeout 300 python tools/c4_kernels.py >> gpurun_out/r3n_ab.log 2>&1
  else STAMG_LIB=abl/$v.so timeout 300 python tools/c4_kernels.py >> gpurun_out/r3n_ab.log 2>&1; fi
done
for v in default sweep_old default sweep_old; do
  if [ "$v" = default ]; then timeout 300 python tools/sweep_ab.py 10 >> gpurun_out/r3n_ab.log 2>&1
  else STAMG_LIB=abl/$v.so timeout 300 python tools/sweep_ab.py 10 >> gpurun_out/r3n_ab.log 2>&1; fi
done
cat gpurun_out/r3n_ab.log

cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -q -x > gpurun_out/r3p_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3p_tests.log
tail -3 gpurun_out/r3p_tests.log
for v in default ms_off ms_all ms_t4 ms_t16 ms_m2 default; do
  echo "== $v" >> gpurun_out/r3p_ab.log
  if [ "$v" = default ]; then timeout 300 python tools/c4_kernels.py >> gpurun_out/r3p_ab.log 2>&1
  else STAMG_LIB=abl/$v.so timeout 300 python tools/c4_kernels.py >> gpurun_out/r3p_ab.log 2>&1; fi
done
cat gpurun_out/r3p_ab.log

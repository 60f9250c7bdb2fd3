cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_shard_sweep.py tests/test_gpu_fullsize_golden.py tests/test_gpu_c4n64_golden.py tests/test_gpu_sharded_emulation.py tests/test_gpu_fold_gate.py tests/test_gpu_fullsize.py -m gpu -q -k "not test_solve or fullsize" > gpurun_out/r2c_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2c_tests.log
for i in 1 2; do
  C5N=512 timeout 600 python tools/perf_probe.py si > gpurun_out/r2c_si_tma_$i.json 2>&1
  STAMG_LIB=abl/gemm_cpasync.so C5N=512 timeout 600 python tools/perf_probe.py si > gpurun_out/r2c_si_cpa_$i.json 2>&1
done
timeout 600 python tools/perf_probe.py c4v > gpurun_out/r2c_c4v_tma.json 2>&1
STAMG_LIB=abl/gemm_cpasync.so timeout 600 python tools/perf_probe.py c4v > gpurun_out/r2c_c4v_cpa.json 2>&1

cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_coarse_chain.py tests/test_gpu_coarse_cluster.py -m gpu -q -x > gpurun_out/r2o_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2o_tests.log
timeout 200 python tools/gs_probe.py 4 10 > gpurun_out/r2o_gs_split.log 2>&1
STAMG_GS_SPLIT=0 timeout 200 python tools/gs_probe.py 4 10 > gpurun_out/r2o_gs_whole.log 2>&1
timeout 200 python tools/gs_probe.py 4 10 64 >> gpurun_out/r2o_gs_split.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_c4n64_golden.py -m gpu -q -x -k "c4 or coarse or mg_apply or gmres" > gpurun_out/r2o_par.log 2>&1; echo "rc=$?" >> gpurun_out/r2o_par.log

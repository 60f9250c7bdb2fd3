cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export STAMG_GS_ROWS_LANES=1
for k in 1 2 3; do timeout 60 python tools/gs_probe.py $k 10 16 >> gpurun_out/r2y_probe16.log 2>&1; echo "rc=$?" >> gpurun_out/r2y_probe16.log; done
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "coarse or mg_apply or gmres" > gpurun_out/r2y_par.log 2>&1; echo "rc=$?" >> gpurun_out/r2y_par.log
for k in 1 2 3; do timeout 60 python tools/gs_probe.py $k 10 >> gpurun_out/r2y_probe.log 2>&1; echo "rc=$?" >> gpurun_out/r2y_probe.log; done

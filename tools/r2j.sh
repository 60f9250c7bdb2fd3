cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_reference_parity.py -m gpu -q > gpurun_out/r2j_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_ref.log
GN=24 timeout 600 python tools/generic_probe.py > gpurun_out/r2j_gen24.json 2>&1
GN=32 GBASIS=0 timeout 600 python tools/generic_probe.py > gpurun_out/r2j_gen32c.json 2>&1

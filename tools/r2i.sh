cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
GN=8 timeout 300 python tools/generic_probe.py > gpurun_out/r2i_gen8.json 2>&1
GN=24 timeout 600 python tools/generic_probe.py > gpurun_out/r2i_gen24.json 2>&1
GN=32 GBASIS=0 timeout 600 python tools/generic_probe.py > gpurun_out/r2i_gen32c.json 2>&1

cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 python tools/pcie_probe.py > gpurun_out/r3c_pcie.log 2>&1
nvidia-smi -q | grep -i -A3 "pci" | head -40 >> gpurun_out/r3c_pcie.log

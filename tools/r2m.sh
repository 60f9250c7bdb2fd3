cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_reference_parity.py -m gpu -q > gpurun_out/r2m_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r2m_ref.log
GN=8 timeout 600 python tools/generic_probe.py > gpurun_out/r2m_gen8.json 2>&1
GN=24 timeout 600 python tools/generic_probe.py > gpurun_out/r2m_gen24.json 2>&1
timeout 1500 python -m pytest tests/test_gpu_c4n64_golden.py -m gpu -q > gpurun_out/r2m_c4n64.log 2>&1; echo "rc=$?" >> gpurun_out/r2m_c4n64.log
for k in apply_L_block sweep_block d2m_block m2d_block coarse_gs_kernel; do
  GN=24 timeout 600 ncu --set full --clock-control none -k regex:$k -s 1 -c 1 -o gpurun_out/r2m_$k python tools/generic_probe.py > gpurun_out/r2m_ncu_$k.log 2>&1
  ncu -i gpurun_out/r2m_$k.ncu-rep --page details > gpurun_out/r2m_${k}_details.txt 2>/dev/null
  rm -f gpurun_out/r2m_$k.ncu-rep
done

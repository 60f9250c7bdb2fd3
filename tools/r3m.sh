cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r3m_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3m_tests.log
for v in default al_old al_r8 al_r6m3 al_r4m3 sw_breg sw_nst4 sw_nst8 default; do
  echo "== $v" >> gpurun_out/r3m_ab.log
  if [ "$v" = default ]; then timeout 300 python tools/c4_kernels.py >> gpurun_out/r3m_ab.log 2>&1
  else STAMG_LIB=abl/$v.so timeout 300 python tools/c4_kernels.py >> gpurun_out/r3m_ab.log 2>&1; fi
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_kernel|apply_L_ring|m2d_kernel|d2m_kernel" -c 40 -f -o gpurun_out/r3m_c4k python tools/c4_kernels.py > gpurun_out/r3m_ncu.log 2>&1
ncu -i gpurun_out/r3m_c4k.ncu-rep --page details > gpurun_out/r3m_c4k_details.txt 2>/dev/null
ncu -i gpurun_out/r3m_c4k.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active > gpurun_out/r3m_c4k_raw.csv 2>/dev/null
ncu -i gpurun_out/r3m_c4k.ncu-rep --page source --csv -k regex:sweep_kernel -c 1 > gpurun_out/r3m_sweep_source.csv 2>/dev/null
ncu -i gpurun_out/r3m_c4k.ncu-rep --page source --csv -k regex:m2d_kernel > gpurun_out/r3m_m2d_source.csv 2>/dev/null
rm -f gpurun_out/r3m_c4k.ncu-rep
ls -la gpurun_out
cat gpurun_out/r3m_ab.log

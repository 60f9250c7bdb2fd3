cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 python -m pytest tests/test_gpu_coarse_cluster.py tests/test_gpu_shard_sweep.py -m gpu -q -x > gpurun_out/r2f_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_tests.log
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "sweep or apply_L or wavefront or smoother or source" > gpurun_out/r2f_sweeptests.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_sweeptests.log
for i in 1 2; do
for xb in 1 2 4; do STAMG_SWEEP_XB=$xb timeout 300 python tools/sweep_ab.py 10 >> gpurun_out/r2f_sweep_ab.log 2>&1; done
STAMG_SWEEP_XB=1 STAMG_LIB=abl/bulk0.so timeout 300 python tools/sweep_ab.py 10 >> gpurun_out/r2f_sweep_ab.log 2>&1
STAMG_SWEEP_XB=2 STAMG_LIB=abl/bulk0.so timeout 300 python tools/sweep_ab.py 10 >> gpurun_out/r2f_sweep_ab.log 2>&1
done
timeout 300 python tools/gs_probe.py 4 2 > gpurun_out/r2f_gs4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:coarse_gs -c 1 -o gpurun_out/r2f_gs_c4_blk python tools/gs_probe.py 4 1 > gpurun_out/r2f_ncu_blk.log 2>&1
STAMG_GS_CHAIN_BLOCKS=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:coarse_gs -c 1 -o gpurun_out/r2f_gs_c4_seq python tools/gs_probe.py 4 1 > gpurun_out/r2f_ncu_seq.log 2>&1
for v in blk seq; do
  ncu -i gpurun_out/r2f_gs_c4_$v.ncu-rep --page source --csv --print-source sass > gpurun_out/r2f_gs_c4_${v}_source.csv 2>/dev/null
  ncu -i gpurun_out/r2f_gs_c4_$v.ncu-rep --page details > gpurun_out/r2f_gs_c4_${v}_details.txt 2>/dev/null
done
ls -la gpurun_out/*.ncu-rep >> gpurun_out/r2f_gs4.log
rm -f gpurun_out/r2f_gs_c4_seq.ncu-rep gpurun_out/r2f_gs_c4_blk.ncu-rep

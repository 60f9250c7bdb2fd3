# GPU session script (run under gpurun from the repo root); $1 = tag, $2 = mode
set -x
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
T=${1:-run}
MODE=${2:-full}
if [ "$MODE" = full ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_tests.log
  timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
fi
if [ "$MODE" = gsq ]; then
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_tests.log
  for k in 1 2 3 4; do timeout 300 python tools/gs_probe.py $k 10 >> gpurun_out/${T}_gs.log 2>&1; done
  timeout 900 python bench.py --steps 3 --no-si --no-e2e --no-cpu --solve-configs 1 2 3 4 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
fi
if [ "$MODE" = gsab ]; then
  for k in 1 2 3; do timeout 300 python tools/gs_probe.py $k 10 >> gpurun_out/${T}_gs.log 2>&1; done
  for k in 1 2 3; do STAMG_GS_MW=1 timeout 300 python tools/gs_probe.py $k 10 >> gpurun_out/${T}_gs_mw.log 2>&1; done
  STAMG_GS_MW=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "coarse or mg_apply or solve" > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_tests.log
fi
if [ "$MODE" = gsprofmw ]; then
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:coarse_gs -c 1 -o gpurun_out/${T}_gs_c3 python tools/gs_probe.py 3 1 > gpurun_out/${T}_ncu3.log 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:coarse_gs -c 1 -o gpurun_out/${T}_gs_c4 python tools/gs_probe.py 4 1 > gpurun_out/${T}_ncu4.log 2>&1
fi
if [ "$MODE" = gst ]; then
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_fullsize_golden.py -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_tests.log
  for k in 1 2 3 4; do timeout 300 python tools/gs_probe.py $k 10 >> gpurun_out/${T}_gs.log 2>&1; done
fi
if [ "$MODE" = final ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_tests.log
  timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
  timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-si --no-e2e --no-solve --no-kernels --no-cpu > gpurun_out/${T}_ncu_launch.log 2>&1
  C5N=256 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"d2m|m2d|unfold|fold" -c 18 -o gpurun_out/${T}_si256 python tools/perf_probe.py si > gpurun_out/${T}_ncu_si.log 2>&1
  C5N=128 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_kernel" -c 2 -o gpurun_out/${T}_sweep128 python tools/perf_probe.py c5s > gpurun_out/${T}_ncu_sweep.log 2>&1
  timeout 900 python bench.py --steps 3 --no-si --no-e2e --no-cpu --no-kernels --solve-configs 4 > gpurun_out/${T}_bench_c4.json 2> gpurun_out/${T}_bench_c4.err
fi
if [ "$MODE" = quick ]; then
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_tests.log
  timeout 900 python bench.py --steps 3 --no-si --no-e2e --no-cpu --solve-configs 1 2 3 4 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
fi
if [ "$MODE" = gsprof4 ]; then
  timeout 300 python tools/gs_probe.py 4 1 > gpurun_out/${T}_gs.log 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:coarse_gs -c 1 -o gpurun_out/${T}_gs_c4 python tools/gs_probe.py 4 1 > gpurun_out/${T}_ncu.log 2>&1
fi
if [ "$MODE" = e2e ]; then
  timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "sweep_host" > gpurun_out/${T}_e2etest.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_e2etest.log
  for cd in 256 512 1024; do STAMG_E2E_CHUNK_DIRS=$cd timeout 600 python bench.py --steps 3 --no-si --no-solve --no-kernels --no-cpu > gpurun_out/${T}_e2e_$cd.json 2>> gpurun_out/${T}_e2e.err; done
  STAMG_E2E_PIPELINE=0 timeout 600 python bench.py --steps 3 --no-si --no-solve --no-kernels --no-cpu > gpurun_out/${T}_e2e_serial.json 2>> gpurun_out/${T}_e2e.err
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_tests.log
fi
if [ "$MODE" = cl ]; then
  timeout 300 python -m pytest tests/test_gpu_coarse_cluster.py -m gpu -x -q > gpurun_out/${T}_cltest.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_cltest.log
  for k in 1 2 3 4; do timeout 120 python tools/gs_probe.py $k 10 >> gpurun_out/${T}_gs.log 2>&1; done
  for k in 1 2 3; do STAMG_GS_CLUSTER=0 timeout 120 python tools/gs_probe.py $k 10 >> gpurun_out/${T}_gs0.log 2>&1; done
  timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "coarse or mg_apply or gmres or bicgstab" > gpurun_out/${T}_ptest.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_ptest.log
  timeout 600 python bench.py --steps 3 --no-si --no-e2e --no-cpu --no-kernels --solve-configs 1 2 3 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
  STAMG_FOLD_MIN_H=16 timeout 600 python bench.py --steps 3 --no-si --no-e2e --no-cpu --no-kernels --solve-configs 2 3 > gpurun_out/${T}_bench_fold.json 2> gpurun_out/${T}_bench_fold.err; echo "bench rc=$?"
fi
if [ "$MODE" = gsprofcl ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:coarse_gs -c 1 -o gpurun_out/${T}_gs_c3 python tools/gs_probe.py 3 2 > gpurun_out/${T}_ncu3.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:coarse_gs -c 1 -o gpurun_out/${T}_gs_c2 python tools/gs_probe.py 2 2 > gpurun_out/${T}_ncu2.log 2>&1
fi
if [ "$MODE" = gsprof4mw ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:coarse_gs -c 1 -o gpurun_out/${T}_gs_c4 python tools/gs_probe.py 4 1 > gpurun_out/${T}_ncu4.log 2>&1
fi
if [ "$MODE" = c4fold ]; then
  STAMG_FOLD_MIN_H=16 timeout 900 python bench.py --steps 3 --no-si --no-e2e --no-cpu --no-kernels --solve-configs 4 > gpurun_out/${T}_bench_c4fold.json 2> gpurun_out/${T}_bench_c4fold.err
  STAMG_FOLD_MIN_H=16 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "scatter or mg_apply or gmres or smoother" > gpurun_out/${T}_ptest.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_ptest.log
fi
if [ "$MODE" = chain ]; then
  timeout 300 python -m pytest tests/test_gpu_coarse_cluster.py -m gpu -x -q > gpurun_out/${T}_cltest.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_cltest.log
  for k in 1 2 3 4; do timeout 120 python tools/gs_probe.py $k 10 >> gpurun_out/${T}_gs.log 2>&1; done
  timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "coarse or mg_apply or gmres or bicgstab" > gpurun_out/${T}_ptest.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_ptest.log
  STAMG_FOLD_MIN_H=16 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "scatter or mg_apply or smoother" > gpurun_out/${T}_ftest.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_ftest.log
fi
if [ "$MODE" = abgs ]; then
  for r in 1 2 3; do for v in old new; do for k in 1 2 3 4; do
    STAMG_LIB=ablib/lib_$v.so timeout 120 python tools/gs_probe.py $k 10 2>&1 | tail -1 | sed "s/^/$v /" >> gpurun_out/${T}_ab.log
  done; done; done
  timeout 300 python -m pytest tests/test_gpu_coarse_cluster.py -m gpu -x -q > gpurun_out/${T}_cltest.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_cltest.log
fi
if [ "$MODE" = ramp ]; then
  timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "sweep_host" > gpurun_out/${T}_e2etest.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_e2etest.log
  for r in 1 2; do
  timeout 600 python bench.py --steps 3 --no-si --no-solve --no-kernels --no-cpu > gpurun_out/${T}_e2e_ramp$r.json 2>> gpurun_out/${T}_e2e.err
  STAMG_E2E_RAMP=0 timeout 600 python bench.py --steps 3 --no-si --no-solve --no-kernels --no-cpu > gpurun_out/${T}_e2e_flat$r.json 2>> gpurun_out/${T}_e2e.err
  done
  STAMG_E2E_CHUNK_DIRS=1024 timeout 600 python bench.py --steps 3 --no-si --no-solve --no-kernels --no-cpu > gpurun_out/${T}_e2e_ramp1024.json 2>> gpurun_out/${T}_e2e.err
fi
if [ "$MODE" = shard ]; then
  timeout 600 python tools/shard_probe.py > gpurun_out/${T}_shard_default.log 2>&1
fi
if [ "$MODE" = shard2 ]; then
  timeout 600 python tools/shard_probe.py 1 2 4 8 > gpurun_out/${T}_shard_default.log 2>&1
fi
if [ "$MODE" = xblk ]; then
  timeout 300 python -m pytest tests/test_gpu_shard_sweep.py -m gpu -x -q > gpurun_out/${T}_xtest.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_xtest.log
  timeout 600 python tools/shard_probe.py 1 2 4 8 > gpurun_out/${T}_shard.log 2>&1
  STAMG_SWEEP_XBLOCKS=0 timeout 600 python tools/shard_probe.py 8 > gpurun_out/${T}_shard_noxb.log 2>&1
fi
if [ "$MODE" = orbit ]; then
  timeout 600 python -m pytest tests/test_gpu_shard_sweep.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/${T}_test.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_test.log
  timeout 900 python tools/shard_probe.py 1 2 4 8 > gpurun_out/${T}_shard.log 2>&1
fi
if [ "$MODE" = xbab ]; then
  timeout 300 python tools/shard_probe.py 8 > gpurun_out/${T}_xb2.log 2>&1
fi
if [ "$MODE" = ab8 ]; then
  for r in 1 2; do for v in old new; do for k in 1 2 3; do
    STAMG_LIB=ablib/lib_$v.so timeout 120 python tools/gs_probe.py $k 10 2>&1 | tail -1 | sed "s/^/$v /" >> gpurun_out/${T}_ab.log
  done; done; done
  timeout 300 python -m pytest tests/test_gpu_coarse_cluster.py -m gpu -x -q > gpurun_out/${T}_cltest.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_cltest.log
  timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "coarse or mg_apply or gmres or bicgstab" > gpurun_out/${T}_ptest.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_ptest.log
  timeout 600 python bench.py --steps 3 --no-si --no-e2e --no-cpu --no-kernels --solve-configs 1 2 3 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
fi
echo done
if [ "$MODE" = ab ]; then
  # A/B of library variants built by tools/ab_build.py (abl/<name>.so), interleaved; $3 = variant names
  timeout 600 python -m pytest tests/test_golden.py -m gpu -x -q > gpurun_out/${T}_golden.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_golden.log
  for rep in 1 2; do for v in ${3:-base}; do
    echo "== $v rep $rep" >> gpurun_out/${T}_ab.log
    STAMG_LIB=abl/$v.so C5N=${C5N:-512} timeout 300 python tools/perf_probe.py si >> gpurun_out/${T}_ab.log 2>&1
  done; done
fi
if [ "$MODE" = final2 ]; then
  # the final set with size-bounded outputs (gpurun copies back <= 64 MiB): ncu
  # reports are exported to CSV on the box and only kept when small
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_tests.log
  timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
  timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-si --no-e2e --no-solve --no-kernels --no-cpu > gpurun_out/${T}_ncu_launch.log 2>&1
  C5N=256 timeout 900 ncu --set full --clock-control none -k regex:"d2m|m2d|unfold|fold" -c 18 -o /tmp/${T}_si256 python tools/perf_probe.py si > gpurun_out/${T}_ncu_si.log 2>&1
  ncu -i /tmp/${T}_si256.ncu-rep --page raw --csv > gpurun_out/${T}_si256_raw.csv 2>&1
  C5N=128 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_kernel" -c 2 -o /tmp/${T}_sweep128 python tools/perf_probe.py c5s > gpurun_out/${T}_ncu_sweep.log 2>&1
  ncu -i /tmp/${T}_sweep128.ncu-rep --page raw --csv > gpurun_out/${T}_sweep128_raw.csv 2>&1
  ncu -i /tmp/${T}_sweep128.ncu-rep --page details > gpurun_out/${T}_sweep128_details.txt 2>&1
  timeout 900 python bench.py --steps 3 --no-si --no-e2e --no-cpu --no-kernels --solve-configs 4 > gpurun_out/${T}_bench_c4.json 2> gpurun_out/${T}_bench_c4.err
  for rep in 1 2; do for v in ${3:-}; do
    echo "== $v rep $rep" >> gpurun_out/${T}_ab.log
    STAMG_LIB=abl/$v.so C5N=512 timeout 300 python tools/perf_probe.py si >> gpurun_out/${T}_ab.log 2>&1
  done; done
  du -sh gpurun_out
fi
if [ "$MODE" = abk ]; then
  # A/B of library variants on the bench's config-4 kernel roofline section
  for rep in 1 2; do for v in ${3:-}; do
    echo "== $v rep $rep" >> gpurun_out/${T}_abk.log
    STAMG_LIB=abl/$v.so timeout 400 python bench.py --steps 3 --no-si --no-e2e --no-cpu --no-solve >> gpurun_out/${T}_abk.log 2>&1
  done; done
  STAMG_LIB=abl/m2dm3.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -x -q -k "scatter or apply_A or mg_apply or gmres or golden" > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
fi

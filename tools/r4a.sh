cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/r4a_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r4a_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4a_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r4a_smoke.log
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r4a_tests2.log 2>&1; echo "tests rc=$?" >> gpurun_out/r4a_tests2.log
tail -3 gpurun_out/r4a_tests.log; tail -3 gpurun_out/r4a_tests2.log; tail -2 gpurun_out/r4a_smoke.log

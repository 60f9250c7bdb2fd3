cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for i in 1 2; do
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r3k_tests_$i.log 2>&1; echo "tests rc=$?" >> gpurun_out/r3k_tests_$i.log
done

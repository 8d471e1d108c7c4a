cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python -m pytest tests/test_gpu_parity.py -q -x -k "selftest or query" > gpurun_out/tune_tests.log 2>&1
rc=$?
echo "rc=$rc" >> gpurun_out/tune_tests.log
if [ $rc -ne 0 ]; then exit 1; fi
for c in ${CFGS:-0 1 2 3 4}; do NRC_QUERY_CFG=$c timeout 60 python scripts/time_query.py; done > gpurun_out/tune.log 2>&1

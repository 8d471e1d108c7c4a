# quick GPU loop: trace of the training frame, training/parity tests, short bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/trace_train_w.py > gpurun_out/trace_w.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x ${TESTSEL:-} > gpurun_out/gpu_tests.log 2>&1
echo "gpu tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log

cd $GRAFT_REPO_ROOT
python scripts/trace_train_w.py > gpurun_out/trace_adam_w1.txt 2>&1
bash scripts/ab_run.sh > gpurun_out/ab_adam3.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log

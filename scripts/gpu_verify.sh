cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -rs --timeout 900 > gpurun_out/gpu_tests.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log

# GPU pass: new-domain tests first, then the whole -m gpu suite, smoke, a
# short bench line.  Outputs in gpurun_out/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_domain.py -q -rf --timeout 600 > gpurun_out/gpu_domain.log 2>&1
echo "domain rc=$?" >> gpurun_out/gpu_domain.log
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 900 --ignore=tests/test_gpu_domain.py > gpurun_out/gpu_tests.log 2>&1
echo "gpu tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log

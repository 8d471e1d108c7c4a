# Refresh the headline evidence for the current build: GPU suite, smoke, bench (1080p, 4K),
# ncu launch list, ncu --set full of the three kernels, training trace.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs --timeout 900 > gpurun_out/gpu_tests.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --workload 4k --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_4k.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nrc_query_ts_kernel -s 2 -c 1 \
  -o gpurun_out/prof_query -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_query.log 2>&1
for k in "nrc_train_ws_kernel:prof_train_ws" "nrc_adam_w_kernel:prof_adam_w"; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${k%%:*} -s 12 -c 1 \
    -o gpurun_out/${k##*:} -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${k##*:}.log 2>&1
done
timeout 900 python scripts/bench_width.py > gpurun_out/width.jsonl 2>gpurun_out/width.err
timeout 900 python scripts/bench_depth.py > gpurun_out/depth.jsonl 2>gpurun_out/depth.err
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -Iinclude -DNRC_TRACE_FLUSH -o /tmp/libnrc_trace.so paper_2106_12372_b200/csrc/nrc_api.cu
NRC_LIB_VARIANT=/tmp/libnrc_trace.so python scripts/trace_train_w.py > gpurun_out/trace_w.log 2>&1

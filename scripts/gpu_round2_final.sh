# Round-2 evidence, final kernels: GPU tests, smoke, bench (1080p, 4K), ncu
# launch list + full captures, sanitizers, width / depth ablations, C3,
# reference arm, training trace.
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
{
echo "# compute-sanitizer runs on a B200 (scripts/sanitize_smoke.py: query, train_step, train_frame, train_backward/apply, encode, assemble_targets, query_accumulate at width 64 through the split-schedule partials kernel; widths 32/128 and depths 2/8; a batch above one tile per SM (the single-schedule kernel); the fused peer all-reduce path at world 1)"
echo "## synccheck"; timeout 900 compute-sanitizer --tool synccheck --print-limit 5 python scripts/sanitize_smoke.py 2>&1 | grep -E "COMPUTE-SANITIZER|SUMMARY|ok|rror| at " | head -20
echo "## racecheck"; timeout 1500 compute-sanitizer --tool racecheck --print-limit 5 python scripts/sanitize_smoke.py 2>&1 | grep -E "COMPUTE-SANITIZER|SUMMARY|ok|rror|hazard| at " | head -20
echo "## memcheck (NRC_SANITIZE_MIN=1)"; NRC_SANITIZE_MIN=1 timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python scripts/sanitize_smoke.py 2>&1 | grep -E "COMPUTE-SANITIZER|SUMMARY|ok|rror| at " | head -20
} > gpurun_out/sanitizers.txt 2>&1
timeout 900 python scripts/bench_width.py > gpurun_out/width.jsonl 2>gpurun_out/width.err
timeout 900 python scripts/bench_depth.py > gpurun_out/depth.jsonl 2>gpurun_out/depth.err
timeout 900 python scripts/c3_convergence.py --out gpurun_out/c3.json > gpurun_out/c3.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -Iinclude -DNRC_TRACE_FLUSH -o /tmp/libnrc_trace.so paper_2106_12372_b200/csrc/nrc_api.cu
NRC_LIB_VARIANT=/tmp/libnrc_trace.so python scripts/trace_train_w.py > gpurun_out/trace_w.log 2>&1

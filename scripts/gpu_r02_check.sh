cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{
echo "# compute-sanitizer runs on a B200 (scripts/sanitize_smoke.py: query, train_step, train_frame, train_backward/apply, encode, assemble_targets, query_accumulate at width 64 through the split-schedule partials kernel; widths 32/128 and depths 2/8; a batch above one tile per SM (the single-schedule kernel); the fused peer all-reduce path at world 1)"
echo "## synccheck"; timeout 900 compute-sanitizer --tool synccheck --print-limit 5 python scripts/sanitize_smoke.py 2>&1 | grep -E "COMPUTE-SANITIZER|SUMMARY|ok|rror| at " | head -20; echo "rc=$?"
echo "## racecheck"; timeout 1500 compute-sanitizer --tool racecheck --print-limit 5 python scripts/sanitize_smoke.py 2>&1 | grep -E "COMPUTE-SANITIZER|SUMMARY|ok|rror|hazard| at " | head -20; echo "rc=$?"
echo "## memcheck (NRC_SANITIZE_MIN=1)"; NRC_SANITIZE_MIN=1 timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python scripts/sanitize_smoke.py 2>&1 | grep -E "COMPUTE-SANITIZER|SUMMARY|ok|rror| at " | head -20; echo "rc=$?"
} > gpurun_out/sanitizers.txt 2>&1
bash scripts/ab_variants.sh base NRC_ADAM_WARPS=8 > gpurun_out/ab.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -Iinclude -DNRC_TRACE_FLUSH -o /tmp/libnrc_trace.so paper_2106_12372_b200/csrc/nrc_api.cu
NRC_LIB_VARIANT=/tmp/libnrc_trace.so python scripts/trace_train_w.py > gpurun_out/trace_w.log 2>&1

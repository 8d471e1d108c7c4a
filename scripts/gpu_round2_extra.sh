# Round-2 refresh of the secondary evidence: sanitizers, 4K bench line,
# width / depth ablations, C3 convergence, reference arm.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{
echo "# compute-sanitizer runs on a B200 (scripts/sanitize_smoke.py: query, train_step, train_frame, train_backward/apply, encode, assemble_targets, query_accumulate at width 64 through the split-schedule partials kernel; widths 32/128 and depths 2/8; batches above one tile per SM (the single-schedule kernel); the fused peer all-reduce path at world 1)"
echo "## synccheck"; timeout 900 compute-sanitizer --tool synccheck python scripts/sanitize_smoke.py 2>&1 | grep -E "COMPUTE-SANITIZER|SUMMARY|ok|rror" | head -20; echo "rc=$?"
echo "## racecheck"; timeout 1500 compute-sanitizer --tool racecheck python scripts/sanitize_smoke.py 2>&1 | grep -E "COMPUTE-SANITIZER|SUMMARY|ok|rror|hazard" | head -20; echo "rc=$?"
echo "## memcheck (NRC_SANITIZE_MIN=1)"; NRC_SANITIZE_MIN=1 timeout 900 compute-sanitizer --tool memcheck python scripts/sanitize_smoke.py 2>&1 | grep -E "COMPUTE-SANITIZER|SUMMARY|ok|rror" | head -20; echo "rc=$?"
} > gpurun_out/sanitizers.txt 2>&1
timeout 600 python bench.py --workload 4k --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_4k.log 2>&1
timeout 900 python scripts/bench_width.py > gpurun_out/width.jsonl 2>gpurun_out/width.err
timeout 900 python scripts/bench_depth.py > gpurun_out/depth.jsonl 2>gpurun_out/depth.err
timeout 900 python scripts/c3_convergence.py --out gpurun_out/c3.json > gpurun_out/c3.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1

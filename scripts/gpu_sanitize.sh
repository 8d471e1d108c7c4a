# compute-sanitizer synccheck / racecheck / memcheck over scripts/sanitize_smoke.py
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{
echo "## synccheck"; timeout 900 compute-sanitizer --tool synccheck --print-limit 5 python scripts/sanitize_smoke.py 2>&1 | tail -25
echo "## racecheck"; timeout 1500 compute-sanitizer --tool racecheck --print-limit 5 python scripts/sanitize_smoke.py 2>&1 | tail -25
echo "## memcheck (NRC_SANITIZE_MIN=1)"; NRC_SANITIZE_MIN=1 timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python scripts/sanitize_smoke.py 2>&1 | tail -25
} > gpurun_out/sanitizers_full.txt 2>&1

# A/B on the GPU box: global-timer traces of every variants/libnrc_tr_*.so
# (NRC_TRACE_FLUSH builds), interleaved timings (scripts/ab_time.py, 3 rounds)
# of every other variants/libnrc_*.so.  ROUNDS / TESTS=1 (GPU suite on the
# working-tree build) optional.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for so in variants/libnrc_tr_*.so; do
  [ -e "$so" ] || continue
  tag=$(basename $so .so); tag=${tag#libnrc_}
  NRC_LIB_VARIANT=$so timeout 300 python scripts/trace_train_w.py > gpurun_out/trace_$tag.txt 2>&1
done
for round in $(seq 1 ${ROUNDS:-3}); do
  for so in variants/libnrc_*.so; do
    case $so in *libnrc_tr_*) continue;; esac
    tag=$(basename $so .so); NRC_LIB_VARIANT=$so timeout 300 python scripts/ab_time.py "${tag#libnrc_}" 30
  done
done > gpurun_out/ab.jsonl 2>&1
if [ "${TESTS:-0}" = 1 ]; then
  timeout 1200 python -m pytest tests -m gpu -q -x -rs --timeout 900 > gpurun_out/gpu_tests.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/gpu_tests.log
fi

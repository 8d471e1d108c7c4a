# Whole-frame A/B (scripts/ab_frame.py) of every variants/libnrc_*.so, with the
# training frame as a CUDA graph and as stream launches (NRC_TRAIN_GRAPH=0).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for round in 1 2 3; do
  for so in variants/libnrc_*.so; do
    tag=$(basename $so .so); tag=${tag#libnrc_}
    NRC_LIB_VARIANT=$so timeout 300 python scripts/ab_frame.py "$tag" 40
    NRC_TRAIN_GRAPH=0 NRC_LIB_VARIANT=$so timeout 300 python scripts/ab_frame.py "$tag" 40
  done
done > gpurun_out/ab_frame.jsonl 2>&1

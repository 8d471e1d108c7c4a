# Time every variants/libnrc_*.so with scripts/ab_time.py, interleaved, 3 rounds.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for round in 1 2 3; do
  for so in variants/libnrc_*.so; do
    tag=$(basename $so .so); NRC_LIB_VARIANT=$so timeout 300 python scripts/ab_time.py "${tag#libnrc_}" 30
  done
done

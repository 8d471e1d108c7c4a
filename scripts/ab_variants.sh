# A/B: build libnrc variants on the GPU box (same sources, different -D
# defines; "base" = none) into /tmp and time each with scripts/ab_time.py,
# interleaved twice.  Usage: bash scripts/ab_variants.sh "base" "NRC_X" "NRC_Y=2" ...
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in "$@"; do
  defs=""; [ "$v" != "base" ] && for d in $v; do defs="$defs -D$d"; done
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    -Iinclude $defs -o "/tmp/libnrc_$(echo $v | tr ' =' '__').so" paper_2106_12372_b200/csrc/nrc_api.cu || echo "build $v failed"
done
for round in 1 2; do
  for v in "$@"; do
    NRC_LIB_VARIANT="/tmp/libnrc_$(echo $v | tr ' =' '__').so" timeout 300 python scripts/ab_time.py "$v" 30
  done
done

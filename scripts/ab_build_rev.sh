# Build libnrc from a git revision (or the working tree: "wt") into
# variants/libnrc_<name>.so for an A/B on the GPU box (scripts/ab_run.sh).
# Usage: bash scripts/ab_build_rev.sh <name> <rev|wt> [extra nvcc -D flags]
set -e
cd "$(dirname "$0")/.."
name=$1; rev=$2; shift 2
mkdir -p variants
tmp=$(mktemp -d)
if [ "$rev" = "wt" ]; then cp -r paper_2106_12372_b200/csrc include "$tmp/"; else
  mkdir -p "$tmp/csrc" "$tmp/include"
  for f in $(git ls-tree --name-only "$rev" paper_2106_12372_b200/csrc/); do git show "$rev:$f" > "$tmp/csrc/$(basename $f)"; done
  git show "$rev:include/nrc.h" > "$tmp/include/nrc.h"
fi
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -I"$tmp/include" "$@" -o "variants/libnrc_$name.so" "$tmp/csrc/nrc_api.cu"
rm -rf "$tmp"
echo "variants/libnrc_$name.so"

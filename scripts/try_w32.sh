cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cp paper_2106_12372_b200/libnrc.so /tmp/libnrc_orig.so
for f in build/variants/w32_g*.so; do
  cp $f paper_2106_12372_b200/libnrc.so
  echo "== $f"
  timeout 200 python scripts/bench_width.py 2>&1 | grep '"hidden_width": 32'
done > gpurun_out/w32.log 2>&1
cp /tmp/libnrc_orig.so paper_2106_12372_b200/libnrc.so

# time each prebuilt libnrc variant in build/variants/ (diagnostics)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cp paper_2106_12372_b200/libnrc.so /tmp/libnrc_orig.so
for f in build/variants/*.so; do
  cp $f paper_2106_12372_b200/libnrc.so
  echo "== $f"
  timeout 120 python scripts/time_query.py
done > gpurun_out/variants.log 2>&1
cp /tmp/libnrc_orig.so paper_2106_12372_b200/libnrc.so

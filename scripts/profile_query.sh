# ncu --set full of one query launch (1080p) inside the bench frame
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nrc_query_ts_kernel -s 3 -c 1 \
  -o gpurun_out/prof_query_r02 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_query.log 2>&1

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export NRC_QUERY_CFG=${NRC_QUERY_CFG:-0}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:nrc_query_kernel -s 5 -c 1 \
  -o gpurun_out/prof_q -f python scripts/time_query.py > gpurun_out/ncu_q.log 2>&1

cd $GRAFT_REPO_ROOT
bash scripts/ab_run.sh > gpurun_out/ab_g.log 2>&1

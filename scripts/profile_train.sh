# ncu --set full of one partials kernel and one optimiser kernel inside a
# training frame (warm L2: --cache-control none), plus the bench launch list.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on \
  -k regex:"nrc_(train_w|adam_w)_kernel" -s 20 -c 2 \
  -o gpurun_out/prof_train_r02 -f python scripts/trace_train_w.py > gpurun_out/ncu_train.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1

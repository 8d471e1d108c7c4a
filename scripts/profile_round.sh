# Round evidence on one B200: bench line, ncu launch list of the bench frame,
# one ncu --set full capture each of the query, the training partials and
# the optimiser kernel (bench frame, default L2 flush between kernels).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
for k in "nrc_query_ts_kernel:prof_query" "nrc_train_ws_kernel:prof_train_ws" "nrc_adam_w_kernel:prof_adam_w"; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${k%%:*} -s 12 -c 1 \
    -o gpurun_out/${k##*:} -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${k##*:}.log 2>&1
done

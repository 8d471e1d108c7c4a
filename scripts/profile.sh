# Bench line + reference arm + ncu launch list + full captures of the query and
# fused train kernels (1 GPU).  Outputs land in gpurun_out/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
echo "ref rc=$?" >> gpurun_out/bench_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nrc_query_ts_kernel -s 3 -c 1 \
  -o gpurun_out/prof_query -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_query.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nrc_train_kernel -s 3 -c 1 \
  -o gpurun_out/prof_train -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_train.log 2>&1
ls -la gpurun_out

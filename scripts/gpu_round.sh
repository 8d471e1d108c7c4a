# Full GPU pass: tests, smoke, bench line, reference arm, ncu launch list,
# full captures of the query kernel and of the default training kernels,
# width ablation.  Outputs in gpurun_out/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 600 > gpurun_out/gpu_tests.log 2>&1
echo "gpu tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nrc_query_ts_kernel -s 3 -c 1 \
  -o gpurun_out/prof_query -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_query.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nrc_train_w_kernel -s 8 -c 1 \
  -o gpurun_out/prof_train_w -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_train_w.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nrc_adam_w_kernel -s 8 -c 1 \
  -o gpurun_out/prof_adam_w -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_adam_w.log 2>&1
bash scripts/ncu_width.sh
timeout 900 python scripts/c3_convergence.py --out gpurun_out/c3.json > gpurun_out/c3.log 2>&1
ls -la gpurun_out

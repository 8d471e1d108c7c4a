# C4: ncu tensor-pipe utilisation and duration per kernel at each hidden width
# (the last frame of scripts/width_step.py).  Outputs in gpurun_out/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum
for w in 32 64 128; do
  timeout 600 ncu --metrics $M --clock-control none --csv -k regex:nrc_ \
    python scripts/width_step.py $w > gpurun_out/ncu_width_$w.csv 2> gpurun_out/ncu_width_$w.err
done
timeout 600 ncu --metrics $M --clock-control none --csv -k regex:nrc_ \
  python scripts/width_step.py 64 f > gpurun_out/ncu_width_64f.csv 2> gpurun_out/ncu_width_64f.err
timeout 900 python scripts/bench_width.py > gpurun_out/bench_width.jsonl 2> gpurun_out/bench_width.err

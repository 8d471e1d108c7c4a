# A/B of the training kernels (NRC_TRAIN_LEGACY=1: single-schedule kernel), trace, GPU tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do python scripts/ab_time.py ws 30; NRC_TRAIN_LEGACY=1 python scripts/ab_time.py legacy 30; done > gpurun_out/ab.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -Iinclude -DNRC_TRACE_FLUSH -o /tmp/libnrc_trace.so paper_2106_12372_b200/csrc/nrc_api.cu
NRC_LIB_VARIANT=/tmp/libnrc_trace.so python scripts/trace_train_w.py > gpurun_out/trace_w.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 >> gpurun_out/ab.log

"""paper_2106_12372_b200 -- B200-native (sm_100a) hot path of Neural Radiance
Caching (Mueller et al., arXiv 2106.12372): fused encoding + 64-wide MLP query,
fused training step (relative-L2 loss, Adam, EMA), LCG-shuffled frame
training and data-parallel multi-GPU training, behind the C ABI of
include/nrc.h (libnrc.so, built in-tree with nvcc for sm_100a)."""
from .dp import DataParallelFrame, frame_batches, shard
from .nrc import (ADAM_M, ADAM_V, CLAMP_QUERY, EMA_PRINTED_FORM, FACTORIZE, NPARAM, PARAMS_EMA, PARAMS_TRAIN,
                  QUERY_RAW_WEIGHTS, EXACT_ENCODING, Config, NRCError, RadianceCache, lcg_params, selftest_umma, volume_records)

__all__ = ["volume_records", "DataParallelFrame", "frame_batches", "shard", "RadianceCache", "Config", "NRCError", "lcg_params", "selftest_umma", "NPARAM", "FACTORIZE",
           "CLAMP_QUERY", "EMA_PRINTED_FORM", "QUERY_RAW_WEIGHTS", "EXACT_ENCODING", "PARAMS_TRAIN", "PARAMS_EMA", "ADAM_M", "ADAM_V"]

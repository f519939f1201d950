#!/bin/bash
# TS-form component isolation (CGGM_TF32_DEBUG bits: 4 = converters skip the split / stores,
# 8 = drain warps skip the TMEM loads; products are garbage, only the time means anything)
for d in 0 4 8 12; do
  echo "CGGM_TF32_DEBUG=$d"
  CGGM_TF32_DEBUG=$d python tools/gemm_f32_bench.py 2>&1 | grep tf32x3_ts
done

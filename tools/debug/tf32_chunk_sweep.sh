# TS-form chunk length: speed (8192^3 and the FP32 large evaluation) and GEMM accuracy
for ch in 1 2 4 8; do
  echo "ts_chunk=$ch"
  CGGM_TF32_TS_CHUNK=$ch python tools/gemm_f32_bench.py 2>&1 | grep "tf32x3_ts tA=1 tB=0 8192"
  CGGM_TF32_TS_CHUNK=$ch python tools/fp32_bench.py --config large --reps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  large f32', d['f32']['ms'])"
  CGGM_TF32_TS_CHUNK=$ch CGGM_TF32_CHUNK=4 python tools/debug/tf32_acc_probe.py | tail -1
done

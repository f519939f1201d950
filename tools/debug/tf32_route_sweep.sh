# FP32 routing sweep: products with fewer 128x128 tiles than MIN_TILES or K below MIN_K on FFMA
for cfg in "0 0" "0 256" "37 256" "0 512" "0 128" "0 0"; do
  set -- $cfg
  echo "min_tiles=$1 min_k=$2"
  CGGM_TF32_MIN_TILES=$1 CGGM_TF32_MIN_K=$2 python tools/fp32_bench.py --config medium --reps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  medium f32', d['f32']['ms'])"
  CGGM_TF32_MIN_TILES=$1 CGGM_TF32_MIN_K=$2 python tools/fp32_bench.py --config large --reps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  large f32', d['f32']['ms'])"
done

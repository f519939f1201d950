# FP32-variant scheduling knobs at `large` (GPU box; ms per evaluation, 5 reps each)
mkdir -p gpurun_out
run() { echo "$1 :: $(env $1 timeout 240 python tools/fp32_bench.py --only f32 --reps 5 2>&1 | tail -1)"; }
for s in "X=0" "CGGM_SIGMA_REC=0" "CGGM_SIGMA_REC=2048" "CGGM_SIGMA_REC=8192" "CGGM_LA_MIN=128" "CGGM_LA_MIN=512" "CGGM_LA_MIN=1024" "CGGM_BINV=2048" "CGGM_BINV=8192" \
         "CGGM_SMALL_KMAX=512" "CGGM_SMALL_KMAX=2048" "CGGM_TF32_MIN_K=128" "CGGM_PRIO_SCHEME=4,5,0,2,3,1,4,5" \
         "CGGM_OBJ_GATE=2432" "X=0"; do run "$s"; done

# Interleaved-Sigma sweep of the composite evaluation at `large` (GPU box; one line per setting):
# CGGM_SIGMA_REC = the smallest recursion node that splits its Sigma block (0 = one lauum after the
# recursion), CGGM_PRIO_SCHEME's 9th entry = the Sigma stream's priority offset.
mkdir -p gpurun_out
run() { echo "$1 :: $(env $1 timeout 180 python tools/part_times.py --parts newton_eval --reps 5 2>&1 | tail -1)"; }
for s in "CGGM_SIGMA_REC=0" "CGGM_SIGMA_REC=4096" "CGGM_SIGMA_REC=8192" "CGGM_SIGMA_REC=2048" \
         "CGGM_SIGMA_REC=4096 CGGM_PRIO_SCHEME=4,5,1,2,3,0,4,5,5" "CGGM_SIGMA_REC=4096 CGGM_PRIO_SCHEME=4,5,1,2,3,0,4,5,1" \
         "CGGM_SIGMA_REC=1024" "CGGM_SIGMA_REC=0"; do run "$s"; done

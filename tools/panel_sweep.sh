# Recursion split sweep of the composite evaluation at `large` (GPU box): CGGM_SPLIT_PANEL = leading
# panel width of the right-looking recursion (0 = halving), with / without the interleaved Sigma.
mkdir -p gpurun_out
run() { echo "$1 :: $(env $1 timeout 180 python tools/part_times.py --parts newton_eval --reps 5 2>&1 | tail -1)"; }
for s in "CGGM_SPLIT_PANEL=0" "CGGM_SPLIT_PANEL=2048" "CGGM_SPLIT_PANEL=1024" "CGGM_SPLIT_PANEL=3072" "CGGM_SPLIT_PANEL=4096" \
         "CGGM_SPLIT_PANEL=2048 CGGM_SIGMA_REC=0" "CGGM_SPLIT_PANEL=1536" "CGGM_SPLIT_PANEL=0"; do run "$s"; done

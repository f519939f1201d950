# Objective start gate sweep at `large` (CGGM_OBJ_GATE = inverse-recursion column at which the
# objective's trial factorisation may start; 0 = together)
mkdir -p gpurun_out
run() { echo "$1 :: $(env $1 timeout 180 python tools/part_times.py --parts newton_eval --reps 5 2>&1 | tail -1)"; }
for s in "CGGM_OBJ_GATE=0" "CGGM_OBJ_GATE=64" "CGGM_OBJ_GATE=2432" "CGGM_OBJ_GATE=4992" "CGGM_OBJ_GATE=7488" "CGGM_OBJ_GATE=9984" "CGGM_OBJ_GATE=12480" "CGGM_OBJ_GATE=14976" "CGGM_OBJ_GATE=0"; do run "$s"; done

# Programmatic dependent launch on / off (CGGM_PDL) for the composite `large` evaluation
mkdir -p gpurun_out
run() { echo "$1 :: $(env $1 timeout 180 python tools/part_times.py --parts newton_eval --reps 5 2>&1 | tail -1)"; }
for s in "CGGM_PDL=0" "CGGM_PDL=1" "CGGM_PDL=0" "CGGM_PDL=1"; do run "$s"; done

# mid-size products on the 128x64 warp-specialised tiles from N quarter waves (CGGM_MID_MIN_WAVES)
mkdir -p gpurun_out
run() { echo "$1 :: $(env $1 timeout 180 python tools/part_times.py --parts newton_eval --reps 5 2>&1 | tail -1)"; }
for s in "CGGM_MID_MIN_WAVES=0" "CGGM_MID_MIN_WAVES=4" "CGGM_MID_MIN_WAVES=6" "CGGM_MID_MIN_WAVES=8" "CGGM_MID_MIN_WAVES=3" "CGGM_MID_MIN_WAVES=0"; do run "$s"; done

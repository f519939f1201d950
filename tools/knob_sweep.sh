# Scheduling-knob sweep of the composite evaluation at `large` (run on the GPU box; one line per setting).
mkdir -p gpurun_out
run() { echo "$1 :: $(env $1 timeout 120 python tools/part_times.py --parts newton_eval 2>&1 | tail -1)"; }
for s in "X=0" "CGGM_PRIO_SCHEME=4,5,0,2,3,1,4,5" "CGGM_PRIO_SCHEME=4,5,0,1,3,2,4,5" "CGGM_PRIO_SCHEME=4,5,0,2,3,1,3,5" "CGGM_PRIO_SCHEME=4,5,1,2,3,0,5,5" "CGGM_PRIO_SCHEME=4,5,1,3,4,0,2,5" "CGGM_LA_MIN=128" "CGGM_LA_MIN=512" "CGGM_BINV=2048" "CGGM_BINV=8192" "CGGM_SMALL_KMAX=512" "CGGM_SMALL_KMAX=2048" "X=0"; do run "$s"; done

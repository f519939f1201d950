# grad_Lambda / S_Lambda beside X^T E (CGGM_GL_OVERLAP: 0 in line, 1 side stream at the greatest priority, 2 at the least)
mkdir -p gpurun_out
run() { echo "$1 :: $(env $1 timeout 180 python tools/part_times.py --parts newton_eval --reps 5 2>&1 | tail -1)"; }
for s in "CGGM_GL_OVERLAP=0" "CGGM_GL_OVERLAP=1" "CGGM_GL_OVERLAP=2" "CGGM_GL_OVERLAP=0" "CGGM_GL_OVERLAP=1" "CGGM_GL_OVERLAP=2"; do run "$s"; done

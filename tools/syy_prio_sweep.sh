# host-input S_yy stream priority (10th CGGM_PRIO_SCHEME entry, default 2) for the end-to-end evaluation
mkdir -p gpurun_out
base="4,5,1,2,3,0,4,5,3"
for v in 2 5 0 2 5; do echo "syy_prio=$v :: $(CGGM_PRIO_SCHEME=$base,$v timeout 300 python tools/e2e_parts.py 2>&1 | tail -1)"; done

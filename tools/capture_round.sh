#!/bin/bash
# Round evidence on one B200 (run under gpurun from the repo root): the GPU suite, the default bench
# line, the ncu launch list of one composite evaluation, and an ncu --set full capture of the
# dominant launch (X^T E, 40000 x 20000 x 1000, the largest single launch once Sigma is assembled
# inside the recursion; reproduced through cggm_test_gemm).  Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --config sharded --steps 2 --warmup 3 --no-e2e --no-fp32 --no-variants > gpurun_out/bench_sharded.json 2> gpurun_out/bench_sharded.err; echo "sharded rc=$?"
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size --clock-control none \
  --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --part all > gpurun_out/launches.log 2>&1; echo "launches rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_dmma -c 1 \
  -o gpurun_out/dominant_xte python tools/gemm_one.py 1 0 40000 20000 1000 0 1 0 > gpurun_out/dominant.log 2>&1; echo "dominant rc=$?"

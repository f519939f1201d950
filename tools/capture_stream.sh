#!/bin/bash
# Round-2 ncu --set full captures of the HBM / L2-bound kernels of one `large` evaluation (one launch
# each: W = X Theta, R / E, grad_Lambda, the active-set passes, the objective's column partials).
# Run under gpurun from the repo root after capture_round.sh has passed; outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:'k_spmm|k_grad_lambda|k_lam_flags|k_lam_write|k_lam_scan|k_active_vec|k_r_e_from_acc|k_col_partials' \
  -o gpurun_out/stream_kernels python tools/profile_step.py --part all > gpurun_out/stream_kernels.log 2>&1
echo "stream rc=$?"
python tools/ncu_metrics.py gpurun_out/stream_kernels.ncu-rep gpu__time_duration.sum dram__bytes_read.sum \
  dram__bytes_write.sum dram__throughput.avg.pct_of_peak_sustained_elapsed \
  lts__throughput.avg.pct_of_peak_sustained_elapsed sm__throughput.avg.pct_of_peak_sustained_elapsed \
  lts__t_bytes.sum launch__grid_size launch__registers_per_thread > gpurun_out/stream_kernels_summary.txt 2>&1
echo "summary rc=$?"; head -40 gpurun_out/stream_kernels_summary.txt

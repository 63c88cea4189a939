#!/bin/bash
# ncu evidence for the bench configuration (run under gpurun, one GPU).
# 1) plain run must exit 0; 2) launch list with per-kernel device time;
# 3) (FULL=1) full capture of the first fine-level GS sweep (the dominant kernel).
set -u
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.log || exit 1
KERN='regex:^(gs_|ghost_|residual_|restrict_|interp_add|band_|abs_max|scale_kernel|gather_kernel|scatter_kernel|permute_kernel|gemv_)'
ncu --metrics gpu__time_duration.sum --clock-control none -k "$KERN" -c 3000 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
if [ "${FULL:-0}" = "1" ]; then
  ncu --set full --clock-control none --import-source on -k regex:"${GS_KERNEL:-gs_chain_kernel}" -c 1 \
      -o gpurun_out/gs_diag_full $CMD > gpurun_out/ncu_full.log 2>&1
  tail -2 gpurun_out/ncu_full.log
fi
tail -2 gpurun_out/ncu_launch.log

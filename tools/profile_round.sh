#!/bin/bash
# Round evidence (one GPU): bench line, ncu launch list of the bench command,
# one ncu --set full capture of the finest-level GS sweep.  Each ncu pass only
# after the plain command exited 0.
set -u
TAG=${TAG:-r01}
if [ "${BENCH:-1}" = "1" ]; then
  python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.log || exit 1
fi
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/${TAG}_prof_plain.json 2> gpurun_out/${TAG}_prof_plain.log || exit 1
KERN='regex:^(gs_|ghost_|residual_|restrict_|res_restrict|interp_add|band_|abs_max|scale_kernel|gather_kernel|scatter_kernel|permute_kernel|repitch_|gemv_)'
ncu --metrics gpu__time_duration.sum --clock-control none -k "$KERN" -c 3000 --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
if [ "${FULL:-1}" = "1" ]; then
  ncu --set full --clock-control none --import-source on -k regex:"${GS_KERNEL:-gs_chain_kernel}" -c 1 \
      -o gpurun_out/${TAG}_gs_full $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
  tail -n2 gpurun_out/${TAG}_ncu_full.log
fi

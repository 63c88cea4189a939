#!/bin/bash
# Round evidence (one GPU): bench line, ncu launch list of the bench command,
# ncu --set full captures of the finest-level launch of every cycle kernel.
# Each ncu pass only after the plain command exited 0.
set -u
TAG=${TAG:-r02}
if [ "${BENCH:-1}" = "1" ]; then
  python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.log || exit 1
fi
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-bitexact"
$CMD > gpurun_out/${TAG}_prof_plain.json 2> gpurun_out/${TAG}_prof_plain.log || exit 1
KERN='regex:^(gs_|ghost_|residual_|restrict_|res_restrict|interp_add|band_|abs_max|scale_kernel|gather_kernel|scatter_kernel|permute_kernel|repitch_|gemv_|chain_|initial_field)'
ncu --metrics gpu__time_duration.sum --clock-control none -k "$KERN" -c 3000 --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
if [ "${FULL:-1}" = "1" ]; then
  # the dominant kernel with source-level stalls
  ncu --set full --clock-control none --import-source on -k regex:gs_chain_kernel -c 1 \
      -o gpurun_out/${TAG}_gs_full $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
  # the first (= finest-level) launch of the other cycle kernels; the finest interpolation is the
  # fourth of a cycle
  ncu --set full --clock-control none -k 'regex:^(ghost_persistent|ghost_writeback|residual_march3|restrict_interior|residual_ghost_lex|restrict_ghost|band_bfs|band_iter|band_gather)' \
      -c 14 -o gpurun_out/${TAG}_cycle_kernels $CMD > gpurun_out/${TAG}_ncu_cycle.log 2>&1
  ncu --set full --clock-control none -k regex:interp_add4 -s 3 -c 1 -o gpurun_out/${TAG}_interp $CMD \
      > gpurun_out/${TAG}_ncu_interp.log 2>&1
  tail -n2 gpurun_out/${TAG}_ncu_full.log gpurun_out/${TAG}_ncu_cycle.log gpurun_out/${TAG}_ncu_interp.log
fi

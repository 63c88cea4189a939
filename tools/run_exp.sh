TAG=r02 bash tools/profile_round.sh
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-bitexact"
ncu --set full --clock-control none -k 'regex:^(residual_march3|restrict_interior|restrict_ghost)' -c 4 -o gpurun_out/r02_cycle_kernels2 -f $CMD > gpurun_out/r02_ncu_cycle2.log 2>&1
for c in c3 c1 c2d; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-bitexact > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.log; tail -1 gpurun_out/r02_bench_$c.log; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.log; cat gpurun_out/r02_bench_reference.json | cut -c1-400

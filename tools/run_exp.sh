TAG=r02 bash tools/profile_round.sh
for c in c3 c1 c2d; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-bitexact > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.log; tail -1 gpurun_out/r02_bench_$c.log; done
ls -la gpurun_out/r02_*

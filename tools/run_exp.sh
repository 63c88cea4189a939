timeout 1700 python -m pytest tests -m gpu -x -q > gpurun_out/r02_final_gputest.log 2>&1; tail -3 gpurun_out/r02_final_gputest.log
BENCH=1 FULL=0 TAG=r02 bash tools/profile_round.sh
for c in c3 c1 c2d; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-bitexact > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.log; done
python __graft_entry__.py smoke 2>&1 | tail -3

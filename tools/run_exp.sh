timeout 300 python tools/gs_cmp.py c3:128 > gpurun_out/r02w_b.txt 2>&1; head -1 gpurun_out/r02w_b.txt
timeout 300 python tools/gs_cmp.py c3:256 > gpurun_out/r02w_a.txt 2>&1; head -1 gpurun_out/r02w_a.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02w_gputest.log 2>&1; tail -4 gpurun_out/r02w_gputest.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r02w_bench.json 2> gpurun_out/r02w_bench.log; cat gpurun_out/r02w_bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['breakdown_ms_per_cycle'], d['e2e']['value'])"

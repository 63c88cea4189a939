timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.log; tail -1 gpurun_out/r02_bench.json | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['e2e']['value'], d['roofline']['frac'], d['breakdown_ms_per_cycle'], d['parity']['max_rel_diff'])"

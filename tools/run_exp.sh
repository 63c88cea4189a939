timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 900 python bench.py --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r04a_bench.json; python -c "
import json; d=json.load(open('gpurun_out/r04a_bench.json')); print(d['ms_per_step'], d['value'], d['e2e']['value'], d['breakdown_ms_per_cycle'], d['parity']['max_rel_diff'])"
for c in c3 c1; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-bitexact 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['ms_per_step'], d['value'], d['breakdown_ms_per_cycle'])"; done

timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02y_gputest.log 2>&1; tail -5 gpurun_out/r02y_gputest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02y_bench.json 2> gpurun_out/r02y_bench.log; tail -3 gpurun_out/r02y_bench.log; python - <<'PY'
import json
d=json.loads(open('gpurun_out/r02y_bench.json').read())
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['breakdown_ms_per_cycle'], d['e2e']['value'], d['parity'], d['bitexact_path'])
PY

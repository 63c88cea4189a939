timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
timeout 600 python tools/gs_time.py c3:256 5 2
for c in c3 c1 c2d; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-bitexact --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],3), d['breakdown_ms_per_cycle'])"; done

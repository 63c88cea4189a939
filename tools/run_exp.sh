for c in c1 c2d c3 c4; do
  for gsm in 0 1024 2048 4096 8192; do
    echo "== $c ghost_small=$gsm"
    GMG_GHOST_SMALL=$gsm timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --no-bitexact --steps 20 --warmup 5 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['breakdown_ms_per_cycle']['ghost_sweep'])"
  done
done

#!/bin/bash
# GPU iteration loop: parity tests, GS timelines on levels 0/1, short bench.
set -u
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for L in ${TRACE_LEVELS:-0 1}; do
  GMG_GS_TRACE=1 timeout 300 python tools/gs_trace.py c4:512 $L > gpurun_out/trace$L.txt 2>&1
done
if [ "${BENCH:-1}" = "1" ]; then
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.log
  echo "bench=$?"
fi

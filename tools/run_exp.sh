timeout 1700 python -m pytest tests -m gpu -x -q > gpurun_out/r03k_gputest.log 2>&1; tail -5 gpurun_out/r03k_gputest.log

timeout 900 python -m pytest tests/test_gpu_slabs.py -x -q -m gpu > gpurun_out/r02x_slabs.log 2>&1; tail -30 gpurun_out/r02x_slabs.log

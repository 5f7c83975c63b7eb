mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "buddy or config4" > gpurun_out/p36_tests.txt 2>&1

mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "handles or small_every or micro" > gpurun_out/p16_tests.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_bench_contract.py -x -q > gpurun_out/p16_tests2.txt 2>&1
for i in 1 2; do timeout 300 python tools/micro/per_config.py 1 >> gpurun_out/p16_per_config.txt 2>&1; done
timeout 600 python tools/micro/per_config.py 2 4 >> gpurun_out/p16_per_config.txt 2>&1

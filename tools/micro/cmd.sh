HEAP_DEV_LIB=libheap_t_mt.so timeout 300 python tools/micro/micro_probe.py 2 > gpurun_out/micro_probe.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "micro or edge or rebuild or config1 or config2 or best_fit" > gpurun_out/pytest_micro.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_micro.log
timeout 600 python tools/micro/per_config.py 1 2 > gpurun_out/per_config.txt 2>&1

HEAP_DEV_LIB=libheap_t_bt.so timeout 300 python tools/micro/buddy_probe.py > gpurun_out/buddy_probe.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "buddy or BUDDY or config4 or p5 or p9 or edge or extremes" > gpurun_out/pytest_bud.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_bud.log
for i in 1 2; do timeout 600 python tools/micro/per_config.py 4 2>&1 | cut -c1-120; done > gpurun_out/per_config.txt

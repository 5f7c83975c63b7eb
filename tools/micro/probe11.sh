mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "best_fit or config2 or buddy or config4 or small_every or micro or config1" > gpurun_out/p11_tests.txt 2>&1
tools/micro/build_variant.sh bft -DBF_TIMING=1 > gpurun_out/p11_build.txt 2>&1
HEAP_DEV_LIB=libheap_bft.so timeout 300 python tools/micro/bf_probe2.py 24 > gpurun_out/p11_bf.txt 2>&1
tools/micro/build_variant.sh btime -DBUDDY_TIMING=1 >> gpurun_out/p11_build.txt 2>&1
HEAP_DEV_LIB=libheap_btime.so timeout 300 python tools/micro/buddy_probe.py > gpurun_out/p11_buddy.txt 2>&1
timeout 900 python tools/micro/per_config.py 1 2 4 > gpurun_out/p11_per_config.txt 2>&1

mkdir -p gpurun_out
tools/micro/build_variant.sh bft -DBF_TIMING=1 > gpurun_out/p6_build.txt 2>&1
HEAP_DEV_LIB=libheap_bft.so timeout 300 python tools/micro/bf_probe2.py 24 > gpurun_out/p6_bf.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "buddy or config4" > gpurun_out/p6_tests.txt 2>&1
timeout 300 python tools/tag_profile.py 4 16 > gpurun_out/p6_tags4.txt 2>&1
tools/micro/build_variant.sh btime -DBUDDY_TIMING=1 >> gpurun_out/p6_build.txt 2>&1
HEAP_DEV_LIB=libheap_btime.so timeout 300 python tools/micro/buddy_probe.py > gpurun_out/p6_buddy.txt 2>&1

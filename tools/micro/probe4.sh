mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "buddy or config4" > gpurun_out/p4_tests.txt 2>&1
timeout 300 python tools/tag_profile.py 4 16 > gpurun_out/p4_tags4.txt 2>&1
tools/micro/build_variant.sh btime -DBUDDY_TIMING=1 > gpurun_out/p4_build.txt 2>&1
HEAP_DEV_LIB=libheap_btime.so timeout 300 python tools/micro/buddy_probe.py > gpurun_out/p4_buddy.txt 2>&1
tools/micro/build_variant.sh btime2 -DBUDDY_TIMING=2 >> gpurun_out/p4_build.txt 2>&1
HEAP_DEV_LIB=libheap_btime2.so timeout 300 python tools/micro/buddy_probe.py >> gpurun_out/p4_buddy.txt 2>&1

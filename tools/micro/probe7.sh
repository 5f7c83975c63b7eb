mkdir -p gpurun_out
tools/micro/build_variant.sh btime3 -DBUDDY_TIMING=3 > gpurun_out/p7_build.txt 2>&1
HEAP_DEV_LIB=libheap_btime3.so timeout 300 python tools/micro/buddy_probe.py > gpurun_out/p7_buddy.txt 2>&1

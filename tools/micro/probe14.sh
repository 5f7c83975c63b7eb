mkdir -p gpurun_out
tools/micro/build_variant.sh timing -DENGINE_TIMING=1 > gpurun_out/p14_build.txt 2>&1
HEAP_DEV_LIB=libheap_timing.so timeout 400 python tools/engine_probe.py 5 12 > gpurun_out/p14_probe.txt 2>&1
HEAP_ENGINE_WARPS=1 HEAP_DEV_LIB=libheap_timing.so timeout 400 python tools/engine_probe.py 5 12 > gpurun_out/p14_probe1w.txt 2>&1

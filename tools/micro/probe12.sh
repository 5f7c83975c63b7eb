mkdir -p gpurun_out
for i in 1 2; do
timeout 300 python tools/micro/per_config.py 1 >> gpurun_out/p12_per_config.txt 2>&1
HEAP_MICRO_GRAPH=1 timeout 300 python tools/micro/per_config.py 1 >> gpurun_out/p12_per_config.txt 2>&1
done
timeout 300 python tools/micro/per_config.py 4 >> gpurun_out/p12_per_config.txt 2>&1
tools/micro/build_variant.sh btime -DBUDDY_TIMING=1 >> gpurun_out/p12_build.txt 2>&1
HEAP_DEV_LIB=libheap_btime.so timeout 300 python tools/micro/buddy_probe.py > gpurun_out/p12_buddy.txt 2>&1

mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_alloc_levels -s 8 -c 1 -o gpurun_out/p10_levels python tools/tag_profile.py 4 12 > gpurun_out/p10_ncu.log 2>&1
tools/micro/build_variant.sh btime2 -DBUDDY_TIMING=2 > gpurun_out/p10_build.txt 2>&1
HEAP_DEV_LIB=libheap_btime2.so timeout 300 python tools/micro/buddy_probe.py > gpurun_out/p10_buddy.txt 2>&1
tools/micro/build_variant.sh mt -DMICRO_TIMING=1 >> gpurun_out/p10_build.txt 2>&1
HEAP_DEV_LIB=libheap_mt.so timeout 300 python tools/micro/micro_probe.py 1 > gpurun_out/p10_micro.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/p10_launches1.csv python tools/tag_profile.py 1 12 > gpurun_out/p10_ncu1.log 2>&1

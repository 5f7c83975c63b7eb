mkdir -p gpurun_out
for c in 1 2 3 4; do echo "== cfg $c"; timeout 300 python tools/tag_profile.py $c 12; done > gpurun_out/p1_tags.txt 2>&1
tools/micro/build_variant.sh btime -DBUDDY_TIMING=1 > gpurun_out/p1_build.txt 2>&1
HEAP_DEV_LIB=libheap_btime.so timeout 300 python tools/micro/buddy_probe.py > gpurun_out/p1_buddy.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/p1_launches4.csv python tools/tag_profile.py 4 6 > gpurun_out/p1_ncu4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/p1_launches2.csv python tools/tag_profile.py 2 6 > gpurun_out/p1_ncu2.log 2>&1

mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "best_fit or config2 or small_every or buddy or config4" > gpurun_out/p8_tests.txt 2>&1
tools/micro/build_variant.sh bft -DBF_TIMING=1 > gpurun_out/p8_build.txt 2>&1
HEAP_DEV_LIB=libheap_bft.so timeout 300 python tools/micro/bf_probe2.py 24 > gpurun_out/p8_bf.txt 2>&1
timeout 300 python tools/tag_profile.py 2 16 > gpurun_out/p8_tags2.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_alloc_levels -s 8 -c 1 -o gpurun_out/p8_levels python tools/tag_profile.py 4 12 > gpurun_out/p8_ncu.log 2>&1

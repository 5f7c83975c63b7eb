mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_alloc_levels -s 8 -c 1 -o gpurun_out/p21_levels python tools/tag_profile.py 4 12 > gpurun_out/p21_ncu.log 2>&1

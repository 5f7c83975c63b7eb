mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_bf_spec_engine -s 8 -c 1 -o gpurun_out/p38_bf python tools/tag_profile.py 2 12 > gpurun_out/p38_ncu_bf.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_alloc_levels -s 8 -c 1 -o gpurun_out/p38_lv python tools/tag_profile.py 4 12 > gpurun_out/p38_ncu_lv.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_micro_step -s 8 -c 1 -o gpurun_out/p38_ms python tools/micro/per_config.py 1 > gpurun_out/p38_ncu_ms.log 2>&1

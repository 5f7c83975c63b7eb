mkdir -p gpurun_out/prof
ncu --set full --clock-control none -k regex:"k_os_scatter|k_scan_1p|k_os_hist" -s 40 -c 8 -o gpurun_out/prof/freepath_lb python tools/engine_probe.py 5 4 > gpurun_out/prof/lb.log 2>&1
timeout 300 python tools/tag_profile.py 5 8 > gpurun_out/tags5.txt 2>&1
timeout 300 python tools/tag_profile.py 4 12 > gpurun_out/tags4.txt 2>&1

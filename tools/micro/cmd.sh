mkdir -p gpurun_out/prof
ncu --set full --clock-control none --import-source on -k regex:k_micro_alloc -s 12 -c 1 -o gpurun_out/prof/micro_alloc python tools/micro/micro_probe.py 1 > gpurun_out/prof/ma.log 2>&1

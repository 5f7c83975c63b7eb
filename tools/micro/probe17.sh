mkdir -p gpurun_out
for g in 592 148 64 32; do echo "== G=$g" >> gpurun_out/p17_grid.txt; HEAP_GRID=$g timeout 300 python tools/micro/per_config.py 4 3 >> gpurun_out/p17_grid.txt 2>&1; done

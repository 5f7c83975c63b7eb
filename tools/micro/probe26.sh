mkdir -p gpurun_out
HEAP_ENGINE_WARPS=3 timeout 1800 python -m pytest tests -q -m gpu -x -k "tlsf or segfit or config5 or config3 or small_every or wild or engine or hybrid or lifo" > gpurun_out/p26_tests.txt 2>&1
tools/micro/build_variant.sh timing -DENGINE_TIMING=1 > gpurun_out/p26_build.txt 2>&1
for w in 2 3; do echo "== warps $w" >> gpurun_out/p26_probe.txt; HEAP_ENGINE_WARPS=$w HEAP_DEV_LIB=libheap_timing.so timeout 400 python tools/engine_probe.py 5 12 2>&1 | tail -2 >> gpurun_out/p26_probe.txt; done
for w in 2 3; do echo "== warps $w" >> gpurun_out/p26_bench.txt; HEAP_ENGINE_WARPS=$w timeout 900 python bench.py --steps 20 --warmup 5 --no-per-config --no-hybrid --no-driver-baselines --no-e2e >> gpurun_out/p26_bench.txt 2>/dev/null; done

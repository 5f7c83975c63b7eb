mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -x -k "tlsf or segfit or config5 or config3 or small_every or wild or engine or hybrid or smoke or lifo or partial" > gpurun_out/p19_tests.txt 2>&1
tools/micro/build_variant.sh timing -DENGINE_TIMING=1 > gpurun_out/p19_build.txt 2>&1
HEAP_DEV_LIB=libheap_timing.so timeout 400 python tools/engine_probe.py 5 12 > gpurun_out/p19_probe.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-per-config --no-hybrid --no-driver-baselines > gpurun_out/p19_bench.json 2> gpurun_out/p19_bench.err

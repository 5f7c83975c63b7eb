mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small_every or wild or config3 or edge or config5_first or engine" 2>&1 | tail -4 > gpurun_out/par_g.txt
HEAP_DEV_LIB=libheap_t_g.so timeout 300 python tools/engine_probe.py 5 12 2>&1 | tail -2 > gpurun_out/probe_g.txt
HEAP_ENGINE_WARPS=1 HEAP_DEV_LIB=libheap_t_g.so timeout 300 python tools/engine_probe.py 5 12 2>&1 | tail -2 >> gpurun_out/probe_g.txt
timeout 600 python bench.py --steps 20 --warmup 5 2>&1 | tail -1 > gpurun_out/bench_g.txt

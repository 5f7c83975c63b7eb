mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "buddy or config4 or handles" > gpurun_out/p23_tests.txt 2>&1
for i in 1 2; do for L in libheap_base.so libheap.so; do echo "== $L" >> gpurun_out/p23_ab.txt; HEAP_DEV_LIB=$L timeout 300 python tools/micro/per_config.py 4 >> gpurun_out/p23_ab.txt 2>&1; done; done

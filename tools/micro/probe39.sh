mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/p39_tests.txt 2>&1
for i in 1 2; do for L in libheap_base.so libheap.so; do echo "== $L" >> gpurun_out/p39_ab.txt; HEAP_DEV_LIB=$L timeout 400 python tools/micro/per_config.py 4 2 >> gpurun_out/p39_ab.txt 2>&1; done; done

mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "micro or small_every or config1 or handles or first_fit or table_rebuild" > gpurun_out/p37_tests.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/p37_tests_all.txt 2>&1
for i in 1 2 3; do for L in libheap_base.so libheap.so; do echo "== $L" >> gpurun_out/p37_ab.txt; HEAP_DEV_LIB=$L timeout 300 python tools/micro/per_config.py 1 >> gpurun_out/p37_ab.txt 2>&1; done; done

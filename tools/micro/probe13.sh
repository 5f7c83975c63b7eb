mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "best_fit or buddy or config4 or config2" > gpurun_out/p13_tests.txt 2>&1
for i in 1 2; do
for L in libheap_base.so libheap.so; do echo "== $L" >> gpurun_out/p13_ab.txt; HEAP_DEV_LIB=$L timeout 300 python tools/micro/per_config.py 4 2 >> gpurun_out/p13_ab.txt 2>&1; done
done

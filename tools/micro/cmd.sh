for v in t_pf0 t_u4; do echo "== $v"; HEAP_DEV_LIB=libheap_$v.so timeout 300 python tools/engine_probe.py 5 12 2>&1 | tail -3; done > gpurun_out/probe_u4.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small_every_batch or wild or config3 or edge or config5_first or direct or lifo" > gpurun_out/pytest_u4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_u4.log

mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -x -k "small_every or buddy or config4 or config2 or best_fit or handles or tlsf_edge or table_rebuild or partial or hybrid" > gpurun_out/p29_tests.txt 2>&1
for i in 1 2; do for f in 0 1; do echo "== HEAP_FUSED=$f" >> gpurun_out/p29_ab.txt; HEAP_FUSED=$f timeout 400 python tools/micro/per_config.py 4 2 >> gpurun_out/p29_ab.txt 2>&1; done; done

mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "best_fit or config2 or small_every" > gpurun_out/p5_tests.txt 2>&1
for e in 0 3; do echo "== HEAP_BF_FLAT=$e"; HEAP_BF_FLAT=$e timeout 300 python tools/tag_profile.py 2 16 | head -3; done > gpurun_out/p5_tags.txt 2>&1
python tools/micro/bf_probe.py 24 > gpurun_out/p5_bf.txt 2>&1

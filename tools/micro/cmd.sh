timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_os.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_os.log
for c in 1 2 3 4; do echo "== cfg $c"; timeout 300 python tools/tag_profile.py $c 12 2>&1 | tail -14; done > gpurun_out/tags_os.txt 2>&1
timeout 300 python tests/dev/bench_all.py 1 2 3 4 > gpurun_out/bench_os.txt 2>&1

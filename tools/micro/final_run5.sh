# round-2 final measurement (dev script): GPU suite, bench line, reference arm, smoke, ncu launch list, ncu full capture of the engine
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/h5_smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/h5_gpu_tests.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/h5_bench.json 2> gpurun_out/h5_bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/h5_reference.json 2> gpurun_out/h5_reference.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h5_smoke.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/h5_launches.csv python bench.py --steps 2 --warmup 3 --no-per-config --no-hybrid --no-driver-baselines --no-cpu-baseline > gpurun_out/h5_ncu_list.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_engine -s 5 -c 1 -o gpurun_out/h5_engine python bench.py --steps 1 --warmup 5 --no-per-config --no-hybrid --no-driver-baselines --no-cpu-baseline --no-e2e > gpurun_out/h5_ncu_full.log 2>&1

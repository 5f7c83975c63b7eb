set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/warp_lat tools/micro/warp_lat.cu && /tmp/warp_lat > gpurun_out/warp_lat.txt 2>&1
INC=$(python -c "from paper_2405_07079_b200 import _native as n; print(n.nccl_dirs()[0])"); LIBD=$(python -c "from paper_2405_07079_b200 import _native as n; print(n.nccl_dirs()[1])")
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -DENGINE_TIMING=1 -I $INC -o paper_2405_07079_b200/libheap_timing.so paper_2405_07079_b200/csrc/heap.cu -L $LIBD -l:libnccl.so.2 -Xlinker -rpath,$LIBD
HEAP_DEV_LIB=libheap_timing.so timeout 300 python tools/engine_probe.py 5 12 > gpurun_out/probe_base.txt 2>&1

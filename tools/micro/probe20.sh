mkdir -p gpurun_out
export PATH=$PATH:/usr/local/cuda/bin
which compute-sanitizer > gpurun_out/p20_san.txt 2>&1
for m in spec cls buddy step; do for tool in memcheck racecheck synccheck; do
  echo "== $tool $m"; timeout 900 compute-sanitizer --tool $tool python tools/micro/san_case2.py $m > gpurun_out/p20_raw.txt 2>&1; grep -E "ERROR SUMMARY|san case2 ok|Error|rror:" gpurun_out/p20_raw.txt | head -4; tail -2 gpurun_out/p20_raw.txt
done; done >> gpurun_out/p20_san.txt 2>&1

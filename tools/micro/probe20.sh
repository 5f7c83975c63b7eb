mkdir -p gpurun_out
for m in spec cls buddy step; do for tool in memcheck racecheck synccheck; do
  echo "== $tool $m"; timeout 900 compute-sanitizer --tool $tool python tools/micro/san_case2.py $m 2>&1 | grep -E "ERROR SUMMARY|san case2 ok|Error|rror:" | head -4
done; done > gpurun_out/p20_san.txt 2>&1

#!/bin/bash
# compute-sanitizer over the Fibonacci-buddy and partial-free paths (dev; run on a GPU box)
set -u
run() { echo "== $1 $2"; timeout 900 compute-sanitizer --tool $1 python tests/dev/debug_case.py $2 2>&1 | grep -E "SUMMARY|MISMATCH|done|rror" | head -5; }
for tool in memcheck racecheck synccheck initcheck; do run $tool "10 1048576 500 4000"; done
for tool in memcheck racecheck synccheck initcheck; do run $tool "260 1048576 500 4000"; done
echo "== memcheck partial edges (tail frees)"
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "partial_free_edges or partial_free_parity and p4-A65536" 2>&1 | grep -E "SUMMARY|passed|failed" | head -5

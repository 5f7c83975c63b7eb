#!/bin/bash
# compute-sanitizer over the TLSF / SEGFIT engine with the wilderness split (dev; run on a GPU box)
set -u
run() { echo "== $1 $2"; timeout 900 compute-sanitizer --tool $1 python tests/dev/wild_debug.py $2 2>&1 | grep -E "SUMMARY|MISMATCH|rror|split batches" | tail -3; }
for tool in memcheck racecheck synccheck initcheck; do run $tool "4 16777216 2000 16000 4 12 2 5 84 direct"; done
for tool in memcheck racecheck; do run $tool "3 16777216 2000 16000 4 14 2 5 83 direct"; done
# the blocked BEST_FIT engine
for tool in memcheck racecheck synccheck; do run $tool "2 16777216 2000 16000 4 14 2 5 92 direct"; done

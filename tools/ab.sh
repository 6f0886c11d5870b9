#!/bin/bash
# DEBUG helper: A/B of library builds on one box.  usage: bash tools/ab.sh cfg reps lib1 lib2 ...
# ("default" = the in-tree build); prints ms/epoch and kernel ms per library.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
cfg=$1; reps=$2; shift 2
for r in $(seq $reps); do
  for lib in "$@"; do
    if [ "$lib" = default ]; then unset F2V_LIB; else export F2V_LIB=$PWD/$lib; fi
    timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-fast --no-per-step 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms_per_launch'],3))"
  done
done

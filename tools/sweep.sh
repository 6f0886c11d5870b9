#!/bin/bash
# DEBUG helper: parity tests + a bench sweep over tuning environments.
# usage (on the GPU box): bash tools/sweep.sh [config] "ENV=.. ENV=.." ...
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
out=gpurun_out/sweep.txt
cfgname=${1:-c2}; shift
if [ -n "$PYTEST" ]; then
  python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $out
  tail -2 gpurun_out/pytest_gpu.log >> $out
fi
for cfg in "$@"; do
  env $cfg timeout 300 python bench.py --config $cfgname --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.log
  echo "$cfgname $cfg :: $(python -c "import json;d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],3), round(d['roofline']['frac'],3), round(d['e2e']['value']/1e9,3))" 2>&1 | tail -1)" >> $out
done

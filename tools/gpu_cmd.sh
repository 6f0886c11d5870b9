python -m pytest tests/test_gpu_parity.py tests/test_gpu_eval.py tests/test_gpu_walk.py tests/test_gpu_shards.py -x -q > gpurun_out/t_v21.log 2>&1; tail -5 gpurun_out/t_v21.log
python tools/eval_timing.py > gpurun_out/eval_timing.log 2>&1; cat gpurun_out/eval_timing.log
for c in c3 c2 c4 c1; do
for ov in 0 1; do
  if [ $ov = 0 ]; then export F2V_NO_PREP_OVERLAP=1; else unset F2V_NO_PREP_OVERLAP; fi
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-per-step 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c overlap=$ov exact', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms_per_launch'],3), 'fast', round(d['fast']['ms_per_step'],3), round(d['fast']['roofline']['kernel_ms_per_launch'],3))"
done; done > gpurun_out/ab_v21.log 2>&1; cat gpurun_out/ab_v21.log

run() { # cfg envs...
  c=$1; shift
  env "$@" timeout 300 python bench.py --config $c --precision exact --steps 4 --warmup 3 --no-cpu-baseline --no-per-step --no-fast 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c $*', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms_per_launch'],3))"
}
{
run c2 F2V_WINDOW=48 F2V_RECENT=8
run c2 F2V_WINDOW=32 F2V_RECENT=8
run c2 F2V_WINDOW=64 F2V_RECENT=8
run c2 F2V_WINDOW=96 F2V_RECENT=8
run c2 F2V_WINDOW=48 F2V_RECENT=4
run c2 F2V_WINDOW=48 F2V_RECENT=16
run c2 F2V_WINDOW=96 F2V_RECENT=16
run c2 F2V_WINDOW=128 F2V_RECENT=16
run c2 F2V_WINDOW=48 F2V_RECENT=8 F2V_LGROUP=8
run c2 F2V_WINDOW=48 F2V_RECENT=8 F2V_LGROUP=32
run c2 F2V_WINDOW=48 F2V_RECENT=8 F2V_CHUNK=128
run c2 F2V_WINDOW=48 F2V_RECENT=8 F2V_CHUNK=512
run c3 F2V_WINDOW=48 F2V_RECENT=8
run c3 F2V_WINDOW=32 F2V_RECENT=8
run c3 F2V_WINDOW=96 F2V_RECENT=8
run c3 F2V_WINDOW=48 F2V_RECENT=16
run c3 F2V_WINDOW=24 F2V_RECENT=4
} > gpurun_out/sweep_v25.log 2>&1; cat gpurun_out/sweep_v25.log

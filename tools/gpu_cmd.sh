python -m pytest tests/test_gpu_parity.py tests/test_gpu_steps.py tests/test_gpu_shards.py -x -q > gpurun_out/t_v4.log 2>&1; tail -5 gpurun_out/t_v4.log
python bench.py --no-cpu-baseline --no-per-step > gpurun_out/r2_bench_c3_v4.json 2> gpurun_out/r2_bench_c3_v4.err; tail -c 600 gpurun_out/r2_bench_c3_v4.json
for c in c2 c4 c1; do python bench.py --config $c --no-cpu-baseline --no-per-step --no-fast > gpurun_out/r2_bench_${c}_v4.json 2>/dev/null; done

python -m pytest tests/test_gpu_eval.py -x -q > gpurun_out/t_eval.log 2>&1; tail -25 gpurun_out/t_eval.log
python bench.py --no-cpu-baseline --no-per-step --no-fast --steps 5 > gpurun_out/r2_bench_c3_v5.json 2> gpurun_out/r2_bench_c3_v5.err; tail -c 300 gpurun_out/r2_bench_c3_v5.json

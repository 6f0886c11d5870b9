python -m pytest tests -q -m gpu -x > gpurun_out/t_final1.log 2>&1; tail -3 gpurun_out/t_final1.log
python bench.py > gpurun_out/r2_bench_default_v3.json 2> gpurun_out/r2_bench_default_v3.err; tail -c 3000 gpurun_out/r2_bench_default_v3.json

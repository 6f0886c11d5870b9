python -m pytest tests/test_gpu_shards.py -q -k "nccl" > gpurun_out/t_nccl2.log 2>&1; tail -2 gpurun_out/t_nccl2.log
python bench.py > gpurun_out/r2_bench_default_v3.json 2> gpurun_out/r2_bench_default_v3.err; tail -c 400 gpurun_out/r2_bench_default_v3.json
python bench.py --impl reference > gpurun_out/r2_bench_reference_v3.json 2> gpurun_out/r2_bench_reference_v3.err; tail -c 400 gpurun_out/r2_bench_reference_v3.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:epoch_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/r2_c3_exact_v3 python bench.py --precision exact --steps 1 --warmup 3 --no-cpu-baseline --no-fast --no-per-step > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:epoch_kernel --launch-skip 5 --launch-count 1 -o gpurun_out/r2_c3_fast_v3 python bench.py --precision fast --steps 1 --warmup 3 --no-cpu-baseline --no-per-step > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2_c3_launches_v3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-fast --no-per-step > /dev/null 2>&1
ls gpurun_out | grep v3

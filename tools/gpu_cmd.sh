python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_v9.log 2>&1; tail -1 gpurun_out/smoke_v9.log
python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputests_v9.log 2>&1; tail -3 gpurun_out/r2_gputests_v9.log
python bench.py > gpurun_out/r2_bench_default_v9.json 2> gpurun_out/r2_bench_default_v9.err; tail -c 200 gpurun_out/r2_bench_default_v9.json
python bench.py --impl reference > gpurun_out/r2_bench_reference_v9.json 2> gpurun_out/r2_bench_reference_v9.err
for c in c1 c2 c4; do python bench.py --config $c --no-cpu-baseline > gpurun_out/r2_bench_${c}_v9.json 2> gpurun_out/r2_bench_${c}_v9.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2_c3_launches_v9.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-fast --no-per-step > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:epoch_kernel --launch-skip 5 --launch-count 1 -o gpurun_out/r2_c3_fast_v9 python bench.py --precision fast --steps 1 --warmup 3 --no-cpu-baseline --no-per-step > /dev/null 2>&1
ls gpurun_out | grep v9

set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py --config c3 --precision exact --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c3_exact.json 2> gpurun_out/c3_exact.err
python bench.py --config c3 --precision fast --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c3_fast.json 2> gpurun_out/c3_fast.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:epoch_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/r2_c3_exact_v0 python bench.py --config c3 --precision exact --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c3_exact.log 2>&1
echo done

set -x
python -m pytest tests/test_gpu_parity.py -x -q -k "exact and not full_size" 2>&1 | tail -5
python -m pytest tests/test_gpu_parity.py -x -q -k "full_size_config3" 2>&1 | tail -5
python bench.py --config c3 --precision exact --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c3_exact_v1.json 2> gpurun_out/c3_exact_v1.err
tail -c 1500 gpurun_out/c3_exact_v1.json
echo done

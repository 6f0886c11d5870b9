python tools/eval_timing.py > gpurun_out/eval_timing.log 2>&1; cat gpurun_out/eval_timing.log
F2V_RUN_C5=1 timeout 2400 python -m pytest tests/test_gpu_c5.py -x -q -s > gpurun_out/r2_c5_parity_v6.log 2>&1; tail -15 gpurun_out/r2_c5_parity_v6.log

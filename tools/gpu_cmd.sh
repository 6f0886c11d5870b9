python -m pytest tests -q -m gpu -x -k "not full_size" > gpurun_out/t_all.log 2>&1; tail -3 gpurun_out/t_all.log
python -m pytest tests/test_gpu_steps.py -q -m gpu -s -k "full_size" > gpurun_out/t_full.log 2>&1; tail -3 gpurun_out/t_full.log; grep "sampled steps" gpurun_out/t_full.log

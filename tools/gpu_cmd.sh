python -m pytest tests/test_gpu_shards.py -q -m gpu -x -k "nccl_allgather_library" > gpurun_out/t_nccl.log 2>&1; tail -15 gpurun_out/t_nccl.log

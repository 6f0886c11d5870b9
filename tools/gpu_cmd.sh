for v in "" _inl _reuse2 _reuse3; do
  F2V_LIB=$PWD/paper_2009_10035_b200/lib/libf2v_b200$v.so python bench.py --config c3 --precision exact --steps 3 --warmup 3 --no-cpu-baseline --no-per-step --no-fast > gpurun_out/ab6$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab6$v.json').read().strip().splitlines()[-1]);print('c3 exact $v', d['ms_per_step'], d['roofline']['kernel_ms_per_launch'])"
done
python -m pytest tests/test_gpu_parity.py -q -x -k "pair_golden or config1 or full_size_config3_epoch" 2>&1 | tail -2

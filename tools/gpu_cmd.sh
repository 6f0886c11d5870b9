python -m pytest tests -q -m gpu -x -k "not full_size" > gpurun_out/t_all2.log 2>&1; tail -3 gpurun_out/t_all2.log
python -m pytest tests -q -m gpu -x -k "full_size_config3" -s > gpurun_out/t_c3.log 2>&1; tail -3 gpurun_out/t_c3.log; grep "sampled" gpurun_out/t_c3.log
for v in "" _rm3; do
  F2V_LIB=$PWD/paper_2009_10035_b200/lib/libf2v_b200$v.so python bench.py --config c3 --precision exact --steps 3 --warmup 3 --no-cpu-baseline --no-per-step --no-fast > gpurun_out/ab5$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab5$v.json').read().strip().splitlines()[-1]);print('c3 $v', d['ms_per_step'], d['roofline']['kernel_ms_per_launch'])"
done

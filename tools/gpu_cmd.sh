for r in 1 2; do for lib in default paper_2009_10035_b200/lib/libf2v_b200_p64.so paper_2009_10035_b200/lib/libf2v_b200_p128.so paper_2009_10035_b200/lib/libf2v_b200_p512.so; do
  if [ "$lib" = default ]; then unset F2V_LIB; else export F2V_LIB=$PWD/$lib; fi
  for c in c2 c3; do
  timeout 300 python bench.py --config $c --precision exact --steps 5 --warmup 3 --no-cpu-baseline --no-per-step 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib $c exact', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms_per_launch'],3), 'fast', round(d['fast']['ms_per_step'],3), round(d['fast']['roofline']['kernel_ms_per_launch'],3))"
  done
done; done > gpurun_out/ab_v37.log 2>&1; cat gpurun_out/ab_v37.log

bash tools/ab.sh c3 2 default paper_2009_10035_b200/lib/libf2v_b200_xpf0.so > gpurun_out/ab_v8.log 2>&1; cat gpurun_out/ab_v8.log

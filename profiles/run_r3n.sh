mkdir -p gpurun_out
RR_AB_REPS=4 python profiles/ab_time.py c5 paper_1811_05784_b200/libroomray_b200.so build/ab/oct/libroomray_b200.so > gpurun_out/r3n_ab.log 2>&1

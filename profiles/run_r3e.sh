mkdir -p gpurun_out
L="paper_1811_05784_b200/libroomray_b200.so"; for v in m7s8 m7s4 m6s8 m6s0 d5 d7; do L="$L build/ab/$v/libroomray_b200.so"; done
RR_AB_REPS=4 python profiles/ab_time.py c5 $L > gpurun_out/r3e_ab.log 2>&1

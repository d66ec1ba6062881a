mkdir -p gpurun_out
L="paper_1811_05784_b200/libroomray_b200.so"; for v in pf2 pf1 hcs fcg pf2hcs; do L="$L build/ab/$v/libroomray_b200.so"; done
RR_AB_REPS=4 python profiles/ab_time.py c5 $L > gpurun_out/r3i_ab.log 2>&1

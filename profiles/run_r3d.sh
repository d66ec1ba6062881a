mkdir -p gpurun_out
L=""; for v in nohbuf n8 n4 n0 h8 h4 h0; do L="$L build/ab/$v/libroomray_b200.so"; done
RR_AB_REPS=4 python profiles/ab_time.py c5 $L > gpurun_out/r3d_ab.log 2>&1

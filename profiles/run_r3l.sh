mkdir -p gpurun_out
L="paper_1811_05784_b200/libroomray_b200.so"; for v in gst8 gst5 gst6; do L="$L build/ab/$v/libroomray_b200.so"; done
RR_AB_REPS=4 python profiles/ab_time.py c5 $L > gpurun_out/r3l_ab.log 2>&1

mkdir -p gpurun_out
L="build/ab/gst5/libroomray_b200.so"; for v in gst4 gst2 gst0; do L="$L build/ab/$v/libroomray_b200.so"; done
RR_AB_REPS=4 python profiles/ab_time.py c5 $L > gpurun_out/r3m_ab.log 2>&1

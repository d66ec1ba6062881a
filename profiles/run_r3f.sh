mkdir -p gpurun_out
ncu --set full --import-source on -k regex:trace_kernel -c 1 --clock-control none -o gpurun_out/prof_c5_r3f -f python profiles/ncu_trace.py c5 1 8 > gpurun_out/prof_c5_r3f.log 2>&1

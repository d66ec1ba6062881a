mkdir -p gpurun_out
for v in default:paper_1811_05784_b200/libroomray_b200.so nohbuf:build/ab/nohbuf/libroomray_b200.so; do
  RR_LIB_PATH=$(pwd)/${v#*:} ncu --section SpeedOfLight --section Occupancy --section WarpStateStats --section LaunchStats --section MemoryWorkloadAnalysis \
    -k regex:trace_kernel --clock-control none --csv --page details python profiles/ncu_trace.py c5 1 8 > gpurun_out/r3c_${v%%:*}.csv 2> gpurun_out/r3c_${v%%:*}.err
done

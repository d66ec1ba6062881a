#!/bin/bash
# Round-2 captures (run on the GPU box from the repo root):
#   profiles/ncu_trace_<cfg>.csv  raw per-launch DRAM / L2 bytes and duration of the trace
#                                 kernel (read by bench.py's roofline), one trace of the config
#   gpurun_out/launches_<tag>.csv the launch list of `python bench.py --steps 2 --warmup 3`
set -e
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg,smsp__thread_inst_executed_per_inst_executed.ratio
for c in ${CONFIGS:-c5 c3 c2}; do
  ncu --metrics $M -k regex:trace_kernel --clock-control none --csv --page raw --print-units base \
      python profiles/ncu_trace.py $c > gpurun_out/ncu_trace_$c.csv 2> gpurun_out/ncu_trace_$c.err
done
if [ -n "$LAUNCHES" ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$LAUNCHES.csv \
      python bench.py --steps 2 --warmup 3 > gpurun_out/launches_$LAUNCHES.log 2>&1
fi

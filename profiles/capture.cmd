# how profiles/ncu_trace_<cfg>.csv and profiles/r2_launches_c5.csv were made (GPU box, repo root):
CONFIGS="c5 c3 c2" LAUNCHES=r2c bash profiles/capture.sh
# -> gpurun_out/ncu_trace_<cfg>.csv (copied to profiles/), gpurun_out/launches_r2c.csv (-> profiles/r2_launches_c5.csv)

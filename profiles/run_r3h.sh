mkdir -p gpurun_out
python bench.py --config c2 > gpurun_out/r3h_bench_c2.json 2> gpurun_out/r3h_bench_c2.err
python bench.py --config c3 > gpurun_out/r3h_bench_c3.json 2> gpurun_out/r3h_bench_c3.err
python tests/native/c4_timing.py > gpurun_out/r3h_c4.log 2>&1
RR_TIMING=1 python bench.py --config c3 --steps 3 --warmup 3 > gpurun_out/r3h_c3_timing.json 2> gpurun_out/r3h_c3_timing.err

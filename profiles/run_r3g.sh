mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/r3g_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r3g_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r3g_smoke.log 2>&1
python bench.py --impl reference > gpurun_out/r3g_bench_ref.json 2> gpurun_out/r3g_bench_ref.err
python bench.py > gpurun_out/r3g_bench.json 2> gpurun_out/r3g_bench.err
CONFIGS=c5 LAUNCHES=r3g bash profiles/capture.sh

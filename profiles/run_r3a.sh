set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/r3_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r3_gpu_tests.log
python profiles/e2e_stalls.py pinned 12 > gpurun_out/r3_stalls_cache.log 2>&1
RR_BLOCK_CACHE_MB=0 python profiles/e2e_stalls.py pinned 12 > gpurun_out/r3_stalls_nocache.log 2>&1
python bench.py > gpurun_out/r3_bench.json 2> gpurun_out/r3_bench.err
CONFIGS=c5 LAUNCHES=r3 bash profiles/capture.sh

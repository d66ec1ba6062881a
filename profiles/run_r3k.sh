mkdir -p gpurun_out
python -m pytest tests/test_gpu_default_path.py tests/test_gpu_w8_variants.py tests/test_gpu_wide.py tests/test_gpu_configs.py tests/test_gpu_checked.py -x -q > gpurun_out/r3k_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3k_tests.log
RR_AB_REPS=4 python profiles/ab_time.py c5 paper_1811_05784_b200/libroomray_b200.so > gpurun_out/r3k_ab.log 2>&1

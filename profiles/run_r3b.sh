mkdir -p gpurun_out
python -m pytest tests/test_gpu_default_path.py tests/test_gpu_w8_variants.py tests/test_gpu_wide.py tests/test_gpu_block_cache.py tests/test_gpu_checked.py -x -q > gpurun_out/r3b_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3b_tests.log
RR_AB_REPS=5 python profiles/ab_time.py c5 paper_1811_05784_b200/libroomray_b200.so build/ab/nohbuf/libroomray_b200.so build/ab/sms11/libroomray_b200.so build/ab/hbuf12/libroomray_b200.so > gpurun_out/r3b_ab.log 2>&1

mkdir -p gpurun_out
(df -T / /tmp /var/tmp /dev/shm . ; mount | head -30) > gpurun_out/dio_fs.txt 2>&1
python -m pytest tests/test_gpu_direct_io.py -q -rs -x > gpurun_out/dio_tests.log 2>&1; echo "rc=$?" >> gpurun_out/dio_tests.log
python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_filedma.py -q -x > gpurun_out/dio_reg.log 2>&1; echo "rc=$?" >> gpurun_out/dio_reg.log
tail -3 gpurun_out/dio_tests.log gpurun_out/dio_reg.log

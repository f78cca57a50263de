mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_a2a_chunks.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r02v_t1.txt 2>&1; echo "t1 rc=$?" >> gpurun_out/r02v_t1.txt
tail -15 gpurun_out/r02v_t1.txt

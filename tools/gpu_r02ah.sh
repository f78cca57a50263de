mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_backward.py tests/test_gpu_determinism.py tests/test_gpu_fullsize_bwd.py -q -x > gpurun_out/r02ah_t.txt 2>&1; echo "rc=$?" >> gpurun_out/r02ah_t.txt; tail -2 gpurun_out/r02ah_t.txt
timeout 900 python tools/time_bwd.py 32768 131072 > gpurun_out/r02ah_bwd.txt 2>&1
BWD_DET=1 timeout 900 python tools/time_bwd.py 32768 131072 >> gpurun_out/r02ah_bwd.txt 2>&1; cat gpurun_out/r02ah_bwd.txt

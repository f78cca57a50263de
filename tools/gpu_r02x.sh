mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_backward.py -q -x -k "fused" > gpurun_out/r02x_t1.txt 2>&1; echo "t1 rc=$?" >> gpurun_out/r02x_t1.txt
tail -3 gpurun_out/r02x_t1.txt
timeout 600 python tools/time_bwd.py 32768 131072 > gpurun_out/r02x_bwd.txt 2>&1; cat gpurun_out/r02x_bwd.txt | tail -2
USP_BWD_FUSED_CLUSTER=0 USPB_LIB_PATH=$PWD/paper_2405_07719_b200/libusp_b200_dev.so timeout 600 python tools/time_bwd.py 32768 131072 > gpurun_out/r02x_bwd_nocl.txt 2>&1; cat gpurun_out/r02x_bwd_nocl.txt | tail -2
USPB_LIB_PATH=$PWD/paper_2405_07719_b200/libusp_b200_trace.so timeout 300 python tools/trace_fused.py 32768 > gpurun_out/r02x_trace.txt 2>&1; tail -7 gpurun_out/r02x_trace.txt

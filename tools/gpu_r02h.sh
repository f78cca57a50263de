mkdir -p gpurun_out
USPB_LIB_PATH=$PWD/paper_2405_07719_b200/libusp_b200_trace.so USP_FA_TRACE=1 timeout 300 python tools/trace_fa.py 32768 > gpurun_out/r02h_trace.txt 2>&1
USPB_LIB_PATH=$PWD/paper_2405_07719_b200/libusp_b200_trace.so USP_FA_TRACE=1 timeout 300 python tools/trace_fa.py 131072 > gpurun_out/r02h_trace128.txt 2>&1
tail -6 gpurun_out/r02h_trace.txt gpurun_out/r02h_trace128.txt

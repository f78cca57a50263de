mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -k "rescale or parity or fullsize" > gpurun_out/r02i_gpu_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/r02i_gpu_tests.txt
tail -2 gpurun_out/r02i_gpu_tests.txt
AB_ROUNDS=2 timeout 1500 python tools/ab_fwd.py "" nodefer > gpurun_out/r02i_ab.txt 2>&1
USPB_LIB_PATH=$PWD/paper_2405_07719_b200/libusp_b200_trace.so USP_FA_TRACE=1 timeout 300 python tools/trace_fa.py 32768 > gpurun_out/r02i_trace.txt 2>&1
cut -c1-200 gpurun_out/r02i_ab.txt; tail -5 gpurun_out/r02i_trace.txt

mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -k "rescale or parity" > gpurun_out/r02d_gpu_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/r02d_gpu_tests.txt
tail -3 gpurun_out/r02d_gpu_tests.txt
AB_ROUNDS=2 timeout 1200 python tools/ab_fwd.py "" r01 > gpurun_out/r02d_ab.txt 2>&1
USPB_LIB_PATH=$PWD/paper_2405_07719_b200/libusp_b200_trace.so USP_FA_TRACE=1 timeout 300 python tools/trace_fa.py 32768 > gpurun_out/r02d_trace.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:row_permute --csv --log-file gpurun_out/r02d_reshard_ncu.csv python tools/time_reshard.py > gpurun_out/r02d_reshard_under_ncu.txt 2>&1
cat gpurun_out/r02d_ab.txt | cut -c1-300; tail -5 gpurun_out/r02d_trace.txt

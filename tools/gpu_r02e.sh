mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -k "parity or p2p or rescale or backward" > gpurun_out/r02e_gpu_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/r02e_gpu_tests.txt
tail -3 gpurun_out/r02e_gpu_tests.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"reshard|row_permute" --csv --log-file gpurun_out/r02e_reshard_ncu.csv python tools/time_reshard.py > gpurun_out/r02e_reshard_under_ncu.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"cudnn|sm100|fmha|flash" -c 1 -o gpurun_out/r02e_cudnn python tools/profile_cudnn.py 32768 > gpurun_out/r02e_cudnn_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_fwd -s 1 -c 1 -o gpurun_out/r02e_fa python tools/profile_target.py 32768 2 > gpurun_out/r02e_fa_ncu.log 2>&1
tail -3 gpurun_out/r02e_cudnn_ncu.log gpurun_out/r02e_fa_ncu.log

mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -k "rescale or parity or p2p or backward or nccl or host" > gpurun_out/r02c_gpu_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/r02c_gpu_tests.txt
timeout 600 python tools/time_reshard.py > gpurun_out/r02c_reshard.txt 2>&1
timeout 1500 python tools/ceiling.py > gpurun_out/r02c_ceiling.txt 2>&1
tail -c 1500 gpurun_out/r02c_gpu_tests.txt; cat gpurun_out/r02c_reshard.txt gpurun_out/r02c_ceiling.txt | cut -c1-400

mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/r02b_gpu_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/r02b_gpu_tests.txt
timeout 900 python tools/overlap_nccl.py > gpurun_out/r02b_overlap.txt 2> gpurun_out/r02b_overlap.err
tail -c 2500 gpurun_out/r02b_gpu_tests.txt; tail -3 gpurun_out/r02b_overlap.txt

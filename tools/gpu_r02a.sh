mkdir -p gpurun_out
set -x
python -m pytest tests -m gpu -x -q -k "rescale or parity or host_path or p2p" > gpurun_out/r02a_gpu_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/r02a_gpu_tests.txt
python bench.py --steps 10 --warmup 3 > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err
USP_BENCH_SAME_DEVICE=1 timeout 600 python bench.py --gpus 4 --steps 3 --warmup 3 --skip-e2e > gpurun_out/r02a_bench_same4.json 2> gpurun_out/r02a_bench_same4.err
tail -c 3000 gpurun_out/r02a_gpu_tests.txt

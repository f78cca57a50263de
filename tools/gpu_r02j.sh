mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/r02j_gpu_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/r02j_gpu_tests.txt
tail -3 gpurun_out/r02j_gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02j_smoke.txt 2>&1; echo "smoke rc=$?"
python bench.py --steps 10 --warmup 3 > gpurun_out/r02j_bench.json 2> gpurun_out/r02j_bench.err
head -c 600 gpurun_out/r02j_bench.json
timeout 900 python tools/time_bwd.py > gpurun_out/r02j_bwd.txt 2>&1; tail -5 gpurun_out/r02j_bwd.txt

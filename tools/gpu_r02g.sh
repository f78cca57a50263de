mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/r02g_gpu_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/r02g_gpu_tests.txt
tail -3 gpurun_out/r02g_gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02g_smoke.txt 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err
AB_BWD=1 AB_ROUNDS=2 AB_SHAPES=long timeout 1200 python tools/ab_fwd.py "" bwdf2fp > gpurun_out/r02g_ab_bwd.txt 2>&1
USPB_LIB_PATH=$PWD/paper_2405_07719_b200/libusp_b200_trace.so USP_FA_TRACE=1 timeout 300 python tools/trace_fa.py 32768 > gpurun_out/r02g_trace.txt 2>&1
cat gpurun_out/r02g_ab_bwd.txt | cut -c1-250; tail -4 gpurun_out/r02g_trace.txt; head -c 400 gpurun_out/r02g_bench.json

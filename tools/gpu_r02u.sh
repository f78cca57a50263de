mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/r02u_gpu_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/r02u_gpu_tests.txt
tail -3 gpurun_out/r02u_gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02u_smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02u_smoke.txt
timeout 900 python tools/time_bwd.py > gpurun_out/r02u_bwd.txt 2>&1; tail -3 gpurun_out/r02u_bwd.txt
BWD_DET=1 timeout 900 python tools/time_bwd.py 131072 > gpurun_out/r02u_bwd_det.txt 2>&1; tail -1 gpurun_out/r02u_bwd_det.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 1 -c 1 -o gpurun_out/r02u_fused python tools/profile_bwd.py 32768 2 > gpurun_out/r02u_ncu.log 2>&1; tail -1 gpurun_out/r02u_ncu.log

#!/bin/bash
# Round-2 measurement set (TAG=r02...): GPU suite, smoke, bench line, the
# reference arm, the ncu launch list of the bench command, one ncu --set full
# capture of the forward kernel at 128K, backward timings (fused and
# deterministic).
TAG=${TAG:-r02f}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gpu_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/${TAG}_gpu_tests.txt
tail -2 gpurun_out/${TAG}_gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
head -c 300 gpurun_out/${TAG}_bench.json; echo
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_bench_reference.json 2> gpurun_out/${TAG}_bench_reference.err
head -c 300 gpurun_out/${TAG}_bench_reference.json; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --skip-cpu-baseline --skip-e2e --skip-backward > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_fwd -s 1 -c 1 \
   -o gpurun_out/${TAG}_fa python tools/profile_target.py 131072 2 > gpurun_out/${TAG}_ncu_fa.log 2>&1
tail -1 gpurun_out/${TAG}_ncu_fa.log
timeout 900 python tools/time_bwd.py > gpurun_out/${TAG}_bwd.txt 2>&1
BWD_DET=1 timeout 900 python tools/time_bwd.py 131072 >> gpurun_out/${TAG}_bwd.txt 2>&1
tail -4 gpurun_out/${TAG}_bwd.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 1 -c 1 \
   -o gpurun_out/${TAG}_bwd_fused python tools/profile_bwd.py 32768 2 > gpurun_out/${TAG}_ncu_bwd.log 2>&1
tail -1 gpurun_out/${TAG}_ncu_bwd.log

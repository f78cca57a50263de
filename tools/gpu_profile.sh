#!/bin/bash
# Runs on the GPU box: bench line + ncu launch list + one full capture of the attention kernel.
set -x
mkdir -p gpurun_out
TAG=${TAG:-r01}
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
tail -c 3000 gpurun_out/bench_${TAG}.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 1 --skip-cpu-baseline --skip-e2e --skip-backward > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_fwd -s 1 -c 1 \
   -o gpurun_out/prof_fa_${TAG} python tools/profile_target.py 131072 2 > gpurun_out/ncu_full_${TAG}.log 2>&1
tail -3 gpurun_out/ncu_full_${TAG}.log
ls -la gpurun_out

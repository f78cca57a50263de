#!/bin/bash
# One ncu --set full capture of the attention kernel at L (default 131072).
TAG=${TAG:-dev}; L=${L:-131072}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_fwd -s 1 -c 1 \
   -o gpurun_out/prof_fa_${TAG} python tools/profile_target.py $L 2 > gpurun_out/ncu_full_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_full_${TAG}.log

#!/bin/bash
# ncu --set full of the solver loop's small kernels (eager loop, steady state): one report each
# usage (on the GPU box): bash tools/ncu_small.sh  -> gpurun_out/small_<kernel>.ncu-rep
for k in ${KERNELS:-reduce_parts_kernel s8_kernel normalize_kernel tsqr_kernel accel_solve_kernel chol_kernel solve_gram_kernel coef_kernel}; do
  CPFIT_EAGER=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:"^$k" --launch-skip ${SKIP:-5} -c 1 \
    -o gpurun_out/small_$k python bench.py --steps 12 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/small_$k.log 2>&1
done

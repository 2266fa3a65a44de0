#!/bin/bash
# One GPU-box pass that regenerates the round's evidence under gpurun_out/:
# gpu tests, smoke, default bench line, per-config bench, the bench command's launch list and
# ncu --set full captures of the dominant kernels at C2 (S pass, M0 pass, fused pass).
set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/ev_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ev_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/ev_bench.log 2>&1
timeout 1200 python tools/bench_configs.py c0 c1 c3 c4 > gpurun_out/ev_configs.log 2>&1
CPFIT_EAGER=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
  --log-file gpurun_out/ev_launches.csv python bench.py --steps 20 --warmup 3 --no-extras --no-cpu-baseline \
  > gpurun_out/ev_ncu_bench.log 2>&1
for k in 5 4 3; do
  KINDS=$k REPS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^(sreg|fiber_ws)" -c 1 \
    -o gpurun_out/ev_kind$k python tools/prof_fiber.py > gpurun_out/ev_ncu_kind$k.log 2>&1
done

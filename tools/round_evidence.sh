#!/bin/bash
# One GPU-box pass that regenerates the round's evidence under gpurun_out/ (prefix $1, default
# r02): gpu tests (BASELINE-scale parity included), smoke, both bench arms at the driver's
# settings, the per-config rates, the bench command's launch list and ncu --set full captures of
# the C2 fibre passes (S pass = the roofline kernel, M0 pass, fused pass) and the C4 sparse MTTKRP.
P=${1:-r02}
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > $O/${P}_tests.log 2>&1; echo "tests rc=$?" >> $O/${P}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${P}_smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > $O/${P}_bench.json 2> $O/${P}_bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/${P}_bench_ref.json 2> $O/${P}_bench_ref.err
timeout 1200 python tools/bench_configs.py c0 c1 c3 c4 > $O/${P}_configs.log 2>&1
CPFIT_EAGER=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
  --log-file $O/${P}_launches.csv python bench.py --steps 20 --warmup 3 --no-extras --no-cpu-baseline \
  > $O/${P}_ncu_bench.log 2>&1
for k in 5 4 3; do
  KINDS=$k REPS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^(sreg|fiber_ws)" -c 1 \
    -o $O/${P}_kind$k python tools/prof_fiber.py > $O/${P}_ncu_kind$k.log 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^sp_mttkrp" --launch-skip 3 -c 1 \
  -o $O/${P}_sparse_c4 python tools/sparse_kernels.py > $O/${P}_ncu_sparse.log 2>&1

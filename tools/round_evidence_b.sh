#!/bin/bash
# Second round-2 evidence pass (prefix $1, default r02b): the GPU suite, smoke, both bench arms at
# the driver's settings, per-config rates, the bench command's launch list, and ncu --set full
# captures of the roofline kernel (C2 S pass) and the kernels changed in this pass (sparse MTTKRP
# and line contractions at C4, the slab M0 pass at C3).
P=${1:-r02b}
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --durations=8 > $O/${P}_tests.log 2>&1; echo "tests rc=$?" >> $O/${P}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${P}_smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > $O/${P}_bench.json 2> $O/${P}_bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/${P}_bench_ref.json 2> $O/${P}_bench_ref.err
timeout 1200 python tools/bench_configs.py c0 c1 c3 c4 > $O/${P}_configs.log 2>&1
CPFIT_EAGER=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
  --log-file $O/${P}_launches.csv python bench.py --steps 20 --warmup 3 --no-extras --no-cpu-baseline \
  > $O/${P}_ncu_bench.log 2>&1
KINDS=5 REPS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^sreg" -c 1 \
  -o $O/${P}_kind5 python tools/prof_fiber.py > $O/${P}_ncu_kind5.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^sp_mttkrp2" --launch-skip 3 -c 1 \
  -o $O/${P}_sparse_c4 python tools/sparse_kernels.py > $O/${P}_ncu_sparse.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"sp_line8" --launch-skip 2 -c 1 \
  -o $O/${P}_line8_c4 python tools/sparse_line.py > $O/${P}_ncu_line8.log 2>&1
CPFIT_EAGER=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"m0slab|fobj" --launch-skip 2 -c 2 \
  -o $O/${P}_slab_c3 python tools/bench_configs.py c3 > $O/${P}_ncu_slab.log 2>&1
for r in kind5 sparse_c4 line8_c4 slab_c3; do
  ncu -i $O/${P}_$r.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    > $O/${P}_${r}_traffic.csv 2>/dev/null
done
tail -3 $O/${P}_tests.log

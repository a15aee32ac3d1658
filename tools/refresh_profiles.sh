#!/bin/bash
# Round-end refresh on the GPU box: GPU tests, smoke, one bench line per config
# (+ the reference arm), ncu launch lists, and --set full captures of the two
# DMMA kernels.  Results land in gpurun_out/ (copy the ones to keep into
# profiles/rNN/).
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
for c in c1 c2 c3 c4 c5; do
  python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; tail -1 gpurun_out/bench_$c.log | cut -c1-160
done
python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-160
for c in c1 c2 c3 c4 c5; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
      --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 2 --warmup 1 \
      > gpurun_out/ncu_$c.log 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:k_leaf_dmma -c 1 \
    -o gpurun_out/prof_dmma_r01 python tools/prof_leaf.py --leaves 148 --reps 1 > gpurun_out/ncu_dmma.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_leaf_apply_dmma -s 2 -c 1 \
    -o gpurun_out/prof_apply_dmma_r01 python tools/prof_apply.py > gpurun_out/ncu_apply.log 2>&1
ls gpurun_out

#!/bin/bash
# Round evidence on one B200 (run under gpurun from the repo root):
# full bench, reference arm, per-config sweep, ncu launch list, ncu --set full of k_fused.
set -u
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_reference.json 2>&1; echo "ref rc=$?"
timeout 600 python tools/bench_configs.py > gpurun_out/configs.txt 2>&1; echo "configs rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --e2e-steps 1 --cpu-seconds 1 --no-power-roof > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 2 -c 1 -f -o gpurun_out/prof \
  python bench.py --n 16777216 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-power-roof > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"

#!/bin/bash
# Round evidence on one B200 (run under gpurun from the repo root): GPU suite,
# smoke, the driver's bench command, reference arm, ncu launch list and
# ncu --set full of k_fused (each ncu command after the same command ran plain).
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
timeout 300 python __graft_entry__.py > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
B2="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-per-config --sustained-seconds 0 --no-multi-driver"
timeout 600 $B2 > gpurun_out/plain_b2.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -c 400 --csv --log-file gpurun_out/launches.csv $B2 > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
B="python bench.py --records 16777216 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-per-config --sustained-seconds 0 --no-multi-driver"
timeout 600 $B > gpurun_out/plain_small.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:k_fused -s 2 -c 1 -f -o gpurun_out/prof_headline $B > gpurun_out/ncu_headline.log 2>&1; echo "ncu full rc=$?"

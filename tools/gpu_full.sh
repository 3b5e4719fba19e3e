#!/bin/bash
# GPU-side: the whole -m gpu suite, ten release-gate runs, the crossover sweep
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_full.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/pytest_full.log | tail -6
pass=0
for i in $(seq 1 10); do
  timeout 300 ./oracle/_ref/release_gate > gpurun_out/gate_run_$i.log 2>&1 && pass=$((pass+1))
done
echo "release gate 9/9 in $pass of 10 runs"
timeout 300 python tools/sweep_probe.py 1 2>&1 | tee gpurun_out/sweep_probe.txt | head -12

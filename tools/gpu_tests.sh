#!/bin/bash
# GPU-side: the whole -m gpu suite (no -x: every failure is listed) + the crossover probe
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q ${1:+-k "$1"} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -12
timeout 300 python tools/sweep_probe.py 1 2>&1 | tee gpurun_out/sweep_probe.txt | head -12

#!/bin/bash
# GPU-side: selected tests (args: pytest -k expression) + one bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x ${1:+-k "$1"} > gpurun_out/pytest_quick.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|Error|error" gpurun_out/pytest_quick.log | tail -8
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1

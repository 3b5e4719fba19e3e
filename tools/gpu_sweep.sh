#!/bin/bash
# GPU-side: the release gate's crossover sweep as the device path times it (criterion 5),
# with per-phase host traces (DDM_TRACE=1) to find host stalls
mkdir -p gpurun_out
DDM_TRACE=1 timeout 600 python tools/sweep_probe.py ${1:-2} > gpurun_out/sweep_probe.txt 2> gpurun_out/sweep_trace.txt
echo rc=$?
cat gpurun_out/sweep_probe.txt
awk '$3+0 > 1.0' gpurun_out/sweep_trace.txt | sort | uniq -c | sort -rn | head -30

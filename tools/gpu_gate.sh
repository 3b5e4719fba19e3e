#!/bin/bash
# GPU-side: the reference release gate 3x + the crossover sweep probe
mkdir -p gpurun_out
for i in 1 2 3; do timeout 600 ./oracle/_ref/release_gate > gpurun_out/gate_$i.log 2>&1; echo "gate $i rc=$?"; grep -E "FAIL|passed" gpurun_out/gate_$i.log; done
timeout 600 python tools/sweep_probe.py 2 2>&1 | tee gpurun_out/sweep_probe.txt | grep -E "sweep|N=256|N=512"

#!/bin/bash
# GPU-side: the f32x2 issue-rate probe, the full GPU test suite, one bench line
mkdir -p gpurun_out
(cd tools/probes && ./f32x2_rate) > gpurun_out/f32x2_rate.txt 2>&1; cat gpurun_out/f32x2_rate.txt
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_px.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_px.log

timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/px_bench.json 2> gpurun_out/px_bench.err
python -c "import json; d=json.load(open('gpurun_out/px_bench.json')); s=d['stages']; print('value %.0f fr/s  ms %.4f  spatial %.4f  temporal %.4f  e2e %.0f' % (d['value'], d['ms_per_step'], s['spatial_ms'], s['temporal_ms'], d['e2e']['value']))"

#!/bin/bash
# GPU-side: parity tests (quiet) + one bench line summary
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err
python -c "import json; d=json.load(open('gpurun_out/bench.json')); s=d['stages']; print('value %.0f fr/s  ms %.3f  spatial %.3f ms (%.0f GB/s)  temporal %.3f ms (%.0f GB/s)  e2e %.0f' % (d['value'], d['ms_per_step'], s['spatial_ms'], s['spatial_GBps'], s['temporal_ms'], s['temporal_GBps'], d['e2e']['value']))"

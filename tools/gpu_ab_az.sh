#!/bin/bash
# A/B of library builds on the fused ring-average configs (tools/bench_configs.py <cfg>az):
#   gpurun -- bash tools/gpu_ab_az.sh "<configs>" <rounds> <lib> [<lib> ...]
cfgs=$1; rounds=$2; shift 2
for r in $(seq $rounds); do
  for lib in "$@"; do
    echo -n "r$r $(basename $lib): "
    DDM_B200_LIB=$PWD/$lib timeout 600 python tools/bench_configs.py $cfgs 2>&1 | grep '^{' | \
      python -c "import json,sys; [print(d['config'], round(d['ms_per_step'],4), round(d['spatial_ms'],4), round(d['temporal_ms'],4), end='; ') for d in map(json.loads, sys.stdin)]; print()"
  done
done

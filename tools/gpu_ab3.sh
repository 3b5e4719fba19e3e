#!/bin/bash
# A/B/C timing of library builds (DDM_B200_LIB), per config, device stages:
#   gpurun -- bash tools/gpu_ab3.sh <tag> "<configs>" <rounds> <lib> [<lib> ...]
tag=$1; cfgs=$2; rounds=$3; shift 3
mkdir -p gpurun_out
for cfg in $cfgs; do
  steps=20; [ $cfg = c3 ] && steps=5; [ $cfg = c4 ] && steps=2
  r_cfg=$rounds; [ $cfg = c4 ] && r_cfg=1
  for r in $(seq $r_cfg); do
    for lib in "$@"; do
      out=gpurun_out/ab_${tag}_${cfg}_${r}_$(basename $lib .so).log
      DDM_B200_LIB=$PWD/$lib timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 \
        --no-cpu-baseline --no-e2e > $out 2>&1
      echo -n "$cfg r$r $(basename $lib): "
      grep '^{' $out | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stages']; print(round(d['ms_per_step'],4), 'spatial', round(s['spatial_ms'],4), 'temporal', round(s['temporal_ms'],4))" || tail -3 $out
    done
  done
done

#!/bin/bash
# A/B of two library builds on a long-sequence config (spatial / temporal split):
#   gpurun -- bash tools/gpu_ab_c4.sh <tag> <lib A> <lib B> [config] [rounds]
tag=$1; a=$2; b=$3; cfg=${4:-c4}; rounds=${5:-2}
mkdir -p gpurun_out
for r in $(seq $rounds); do
  for lib in $a $b; do
    echo -n "$cfg $lib: "
    DDM_B200_LIB=$PWD/$lib timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline \
      --no-e2e > gpurun_out/ab_${tag}_${r}_$(basename $lib).log 2>&1
    grep '^{' gpurun_out/ab_${tag}_${r}_$(basename $lib).log | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), round(d.get('spatial_ms',0),3), round(d.get('temporal_ms',0),3))" \
      || tail -5 gpurun_out/ab_${tag}_${r}_$(basename $lib).log
  done
done

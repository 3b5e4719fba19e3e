#!/bin/bash
# A/B timing of two library builds (DDM_B200_LIB) with the gpu tests on the new one:
#   gpurun -- bash tools/gpu_ablib.sh <tag> <lib A> <lib B> [rounds]
tag=$1; a=$2; b=$3; rounds=${4:-3}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$tag.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_$tag.log
for r in $(seq $rounds); do
  for lib in $a $b; do
    echo -n "$lib: "
    DDM_B200_LIB=$PWD/$lib timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e \
      > gpurun_out/ab_${tag}_$r_$(basename $lib).log 2>&1
    grep '^{' gpurun_out/ab_${tag}_$r_$(basename $lib).log | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d.get('spatial_ms',0),4), round(d.get('temporal_ms',0),4))" \
      || tail -5 gpurun_out/ab_${tag}_$r_$(basename $lib).log
  done
done

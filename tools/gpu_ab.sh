#!/bin/bash
# A/B timing of kernel variants selected by env vars, plus gpu tests (default build and, with
# AB_TEST_ENV, the full gpu suite again under that env) and an optional ncu capture.
#   gpurun -- bash tools/gpu_ab.sh <tag> "<ENV=1 ...>" "<ENV=2 ...>" ...
tag=$1; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$tag.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$tag.log
if [ -n "$AB_TEST_ENV" ]; then
  env $AB_TEST_ENV timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_${tag}_env.log 2>&1
  echo "pytest ($AB_TEST_ENV) rc=$?"; tail -3 gpurun_out/pytest_gpu_${tag}_env.log
fi
for v in "$@"; do
  echo "== variant: $v"
  env $v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1
done
if [ -n "$NCU_KERNEL" ]; then
  env $NCU_ENV timeout 600 ncu --set full --clock-control none --import-source on -k regex:$NCU_KERNEL -s 2 -c 1 \
      -o gpurun_out/full_${NCU_KERNEL}_$tag python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  ncu -i gpurun_out/full_${NCU_KERNEL}_$tag.ncu-rep --page raw --csv > gpurun_out/raw_${NCU_KERNEL}_$tag.csv 2>/dev/null
  ncu -i gpurun_out/full_${NCU_KERNEL}_$tag.ncu-rep --page source --csv > gpurun_out/source_${NCU_KERNEL}_$tag.csv 2>/dev/null
  python tools/ncu_summary.py gpurun_out/raw_${NCU_KERNEL}_$tag.csv
  python tools/sass_profile.py gpurun_out/source_${NCU_KERNEL}_$tag.csv 25
fi

#!/bin/bash
# e2e A/B by env switch: gpu tests, then bench.py (e2e on) under each env, interleaved.
#   gpurun -- bash tools/gpu_e2e_ab.sh <tag> "<ENV=a>" "<ENV=b>" [rounds]
tag=$1; a=$2; b=$3; rounds=${4:-2}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$tag.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_$tag.log
for r in $(seq $rounds); do
  for v in "$a" "$b"; do
    env $v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_${tag}.log 2>&1
    echo -n "$v: "
    grep '^{' gpurun_out/e2e_${tag}.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e'].get('serial', d['e2e']); print(round(d['ms_per_step'],3), round(e['ms_per_step'],2), {k: round(v*1e3,2) for k,v in e['phases_s'].items()})"
  done
done

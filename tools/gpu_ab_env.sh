#!/bin/bash
# GPU-side A/B of environment switches on the bench's device stages:
#   tools/gpu_ab_env.sh "tests-k-expr|none" "ENV1=a ENV2=b" "ENV1=c" ...   ("-" = no env)
mkdir -p gpurun_out
if [ "$1" != "none" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x ${1:+-k "$1"} > gpurun_out/pytest_ab.log 2>&1
  echo "pytest rc=$?"; grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_ab.log | tail -6
fi
shift
for rep in 1 2; do
for cfg in "$@"; do
  envs=""; [ "$cfg" != "-" ] && envs="$cfg"
  env $envs timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/ab.json 2> gpurun_out/ab.err
  python - "$cfg" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
    st = d.get("stages", d)
    print("%-40s ms/step %.4f spatial %.4f temporal %.4f" % (sys.argv[1], d["ms_per_step"], st["spatial_ms"], st["temporal_ms"]))
except Exception as e:
    print(sys.argv[1], "FAILED", e, open("gpurun_out/ab.err").read()[-600:])
PY
done; done

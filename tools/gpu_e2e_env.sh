#!/bin/bash
# GPU-side A/B of environment switches on the bench's e2e (C-ABI ddm::run, pinned host buffers)
#   tools/gpu_e2e_env.sh "ENV=a" "-" ...
mkdir -p gpurun_out
for rep in 1 2; do
for cfg in "$@"; do
  envs=""; [ "$cfg" != "-" ] && envs="$cfg"
  env $envs timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/e2e_ab.json 2> gpurun_out/e2e_ab.err
  python - "$cfg" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/e2e_ab.json").read().strip().splitlines()[-1])
    e = d["e2e"].get("serial", d["e2e"])
    print("%-28s e2e %.2f ms  %s" % (sys.argv[1], e["ms_per_step"], {k: round(v * 1e3, 2) for k, v in e["phases_s"].items()}))
except Exception as ex:
    print(sys.argv[1], "FAILED", ex, open("gpurun_out/e2e_ab.err").read()[-600:])
PY
done; done

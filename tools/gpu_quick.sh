#!/bin/bash
# GPU-side: selected tests (args: pytest -k expression; "none" skips them) + one bench line
# (device stages) + the e2e f64-map step times
mkdir -p gpurun_out
if [ "$1" != "none" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x ${1:+-k "$1"} > gpurun_out/pytest_quick.log 2>&1
  echo "pytest rc=$?"; grep -E "passed|failed|Error|error" gpurun_out/pytest_quick.log | tail -8
fi
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/quick_bench.json 2> gpurun_out/quick_bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/quick_bench.json").read().strip().splitlines()[-1])
st = d["stages"]
print("value %.0f ms/step %.4f spatial %.4f temporal %.4f" % (d["value"], d["ms_per_step"], st["spatial_ms"], st["temporal_ms"]))
e = d["e2e"].get("serial", d["e2e"])
print("e2e %.0f frames/s, %.2f ms; phases %s" % (e["value"], e["ms_per_step"], {k: round(v * 1e3, 3) for k, v in e["phases_s"].items()}))
PY

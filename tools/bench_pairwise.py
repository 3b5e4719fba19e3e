"""Device time of the WITHOUT_FT kernel (timing.step2 of ddm::run) at C2 (512^2 x 1024, f32
spectra, f64 sums): all lags (contiguous range) and the log lag set.

    python tools/bench_pairwise.py [W H N]
"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import ddm_oracle as O  # noqa: E402
from paper_2012_05695_b200 import ddm  # noqa: E402

W, H, N = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (512, 512, 1024)
rng = np.random.default_rng(1)
st = rng.integers(0, 4096, size=(N, H, W), dtype=np.uint16)
for name, lags in (("all", []), ("log", O.log_lags(N))):
    cfg = ddm.RunConfig(algorithm="without_ft", precision="f32", lags=lags, memory_bytes=1 << 40)
    ddm.run(st, cfg)
    t = [ddm.run(st, cfg).timing["step2"] for _ in range(3)]
    print(json.dumps({"lags": name, "W": W, "H": H, "N": N, "pairwise_ms": 1e3 * float(np.median(t))}), flush=True)

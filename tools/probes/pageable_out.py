"""Map download into pageable memory: fresh (np.empty, faults on first touch) vs pre-touched
(np.ones) destination, C2 f32 through ddm_b200_run_u16."""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2012_05695_b200 import ddm  # noqa: E402

W = H = 512
N = 1024
st = np.random.default_rng(1).integers(0, 4000, (N, H, W), dtype=np.uint16)
plane = H * (W // 2 + 1)
L = ddm.lib()
cfg = ddm._config(ddm.RunConfig(precision="f32", memory_bytes=1 << 40), [])
print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
for kind in ("empty", "touched", "empty", "touched"):
    out = np.empty(N * plane) if kind == "empty" else np.ones(N * plane)
    lags = np.zeros(N, np.int64)
    nl = C.c_int64(0)
    cnt, tim = ddm.Counters(), ddm.Timing()
    t0 = time.perf_counter()
    rc = L.ddm_b200_run_u16(ddm._p(st, C.c_uint16), W, H, N, C.c_double(1.0), C.byref(cfg),
                            ddm._p(out, C.c_double), C.c_int64(out.size), ddm._p(lags, C.c_int64),
                            C.byref(nl), C.byref(cnt), C.byref(tim))
    wall = time.perf_counter() - t0
    print(f"{kind:8s} rc={rc} wall {wall*1e3:.1f} ms merge {tim.merge*1e3:.1f} ms "
          f"({out.nbytes/tim.merge/1e9:.1f} GB/s) disk {tim.disk*1e3:.1f} ms", flush=True)

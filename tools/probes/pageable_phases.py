"""Phases of ddm::run with PAGEABLE host buffers (numpy in, numpy map out: the C++ API's
std::vector case), f32, several sizes: how fast the pinned-bounce staging paths go."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2012_05695_b200 import ddm  # noqa: E402

for W, H, N in ((64, 64, 1024), (64, 64, 4096), (256, 256, 1024), (512, 512, 1024)):
    st = np.random.default_rng(1).integers(0, 4000, (N, H, W), dtype=np.uint16)
    for rep in range(3):
        t0 = time.perf_counter()
        a = ddm.run(st, ddm.RunConfig(precision="f32", memory_bytes=1 << 40))
        wall = time.perf_counter() - t0
    t = a.timing
    mb_in, mb_out = st.nbytes / 1e6, a.values.nbytes / 1e6
    print(f"{W}x{H}x{N}: wall {wall*1e3:.2f} ms  disk {t['disk']*1e3:.2f} ({mb_in/max(t['disk'],1e-9)/1e3:.1f} GB/s) "
          f"merge {t['merge']*1e3:.2f} ({mb_out/max(t['merge'],1e-9)/1e3:.1f} GB/s) s1 {t['step1']*1e3:.2f} "
          f"s2 {t['step2']*1e3:.2f} other {t['other']*1e3:.2f} total {t['total']*1e3:.2f}", flush=True)

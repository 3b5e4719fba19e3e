"""Device time of the f64 WITH_FT path (generic Stockham engines) at C1/C2/C5 shapes."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2012_05695_b200 import ddm  # noqa: E402

for W, H, N in ((64, 64, 128), (500, 500, 1000), (512, 512, 1024), (1024, 1024, 2048)):
    fr = torch.randint(100, 3000, (N * H * W,), dtype=torch.int32, device="cuda").to(torch.int16)
    out = torch.empty(N * H * (W // 2 + 1), dtype=torch.float64, device="cuda")
    for prec in ("f64", "f32"):
        for _ in range(2):
            sp, tp, nl = ddm.run_device(fr.data_ptr(), 2, W, H, N, out.data_ptr(), precision=prec, out_f64=True)
        print(f"{W}x{H}x{N} {prec}: spatial {sp:.3f} ms temporal {tp:.3f} ms [{ddm.last_engines()}]", flush=True)
    del fr, out
    torch.cuda.empty_cache()

"""Device time of the WITH_FT path on the other BASELINE.json configs (not the headline bench).

    python tools/bench_configs.py [c1 c3 c4 c5 ...]

Frames are synthetic u16 noise generated on the device (transform cost does not depend on
the pixel values; parity on these shapes is covered by the tests). Map f32 in HBM.
"""
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2012_05695_b200 import ddm  # noqa: E402

CONFIGS = {
    "c1": (64, 64, 128),
    "c2": (512, 512, 1024),
    "c3": (1024, 1024, 2048),
    "c4": (2048, 2048, 4096),
    "c5": (500, 500, 1000),
}


def bench_azimuthal(name, steps=5):
    """run + ring average in one pass (fused where the register engines apply)."""
    W, H, N = CONFIGS[name]
    g = torch.Generator(device="cuda").manual_seed(7)
    frames = torch.randint(100, 3000, (N * H * W,), dtype=torch.int32, device="cuda",
                           generator=g).to(torch.int16)
    cap = int((H * H / 4 + W * W / 4) ** 0.5) + 3
    means = torch.empty(N * cap, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        return ddm.run_azimuthal_device(frames.data_ptr(), 2, W, H, N, means.data_ptr(), cap,
                                        stream=stream.cuda_stream)

    nb, _, _, fused = step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sp, tp = [], []
    e0.record(stream)
    for _ in range(steps):
        _, s_, t_, _ = step()
        sp.append(s_)
        tp.append(t_)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    Q = H * (W // 2 + 1)
    alg = N * (2 * W * H + 16 * Q)     # map bytes ~0: only the ring means leave the kernel
    res = {"config": name + "+azimuthal", "fused": fused, "bins": nb, "ms_per_step": ms,
           "frames_per_s": N / ms * 1e3, "spatial_ms": sum(sp) / steps,
           "temporal_ms": sum(tp) / steps, "algorithmic_GBps": alg / ms / 1e6}
    del frames, means
    torch.cuda.empty_cache()
    return res


def bench(name, steps=5):
    W, H, N = CONFIGS[name]
    plane = H * (W // 2 + 1)
    g = torch.Generator(device="cuda").manual_seed(7)
    frames = torch.randint(100, 3000, (N * H * W,), dtype=torch.int32, device="cuda",
                           generator=g).to(torch.int16)
    out = torch.empty(N * plane, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        return ddm.run_device(frames.data_ptr(), 2, W, H, N, out.data_ptr(), "f32", out_f64=False,
                              stream=stream.cuda_stream)

    step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sp, tp = [], []
    e0.record(stream)
    for _ in range(steps):
        s, t, _ = step()
        sp.append(s)
        tp.append(t)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    Q = plane
    alg = N * (2 * W * H + 16 * Q + 4 * Q)
    res = {"config": name, "W": W, "H": H, "N": N, "ms_per_step": ms, "frames_per_s": N / ms * 1e3,
           "spatial_ms": sum(sp) / steps, "temporal_ms": sum(tp) / steps,
           "algorithmic_GBps": alg / ms / 1e6}
    del frames, out
    torch.cuda.empty_cache()
    return res


if __name__ == "__main__":
    for name in sys.argv[1:] or ["c1", "c5", "c3", "c4"]:
        t0 = time.time()
        try:
            if name.endswith("az"):
                print(json.dumps(bench_azimuthal(name[:-2])), flush=True)
            else:
                print(json.dumps(bench(name)), flush=True)
        except Exception as e:  # report and continue with the next config
            print(json.dumps({"config": name, "error": str(e)[:300]}), flush=True)
        print(f"  ({time.time() - t0:.1f} s)", flush=True)

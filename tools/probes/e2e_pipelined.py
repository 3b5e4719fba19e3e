"""Probe: C2 end to end through the staging-session C-ABI, one session at a time (stage the
pinned u16 stack, run WITH_FT into a pinned f64 map) against two sessions in flight on two host
threads (one stack's map D2H overlapping the next stack's frame H2D: PCIe is full duplex and
the two directions use separate copy engines). Prints ms per stack for each."""
import ctypes as C
import sys
import threading
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2012_05695_b200 import ddm  # noqa: E402

W = H = 512
N = 1024
PLANE = H * (W // 2 + 1)


def one_stack(sess, frames, out):
    lib = ddm.lib()
    ddm._check(lib.ddm_b200_stage_frames(sess._h, C.c_void_p(frames.data_ptr()), 0, N))
    counters, timing = ddm.Counters(), ddm.Timing()
    ddm._check(lib.ddm_b200_run_with_ft(sess._h, None, C.c_int64(0), None, C.c_int64(0),
                                        C.c_void_p(out.data_ptr()), C.c_int64(N * PLANE),
                                        C.byref(counters), C.byref(timing)))


def main(steps=12, inflight_list=(1, 2)):
    rng = np.random.default_rng(5)
    st = rng.integers(0, 4096, size=(N, H, W), dtype=np.uint16)
    results = {}
    for inflight in inflight_list:
        sess = [ddm.Session(W, H, N, "f32", 0) for _ in range(inflight)]
        frames = [torch.from_numpy(st).pin_memory() for _ in range(inflight)]
        outs = [torch.empty(N * PLANE, dtype=torch.float64).pin_memory() for _ in range(inflight)]
        for i in range(inflight):
            for _ in range(2):
                one_stack(sess[i], frames[i], outs[i])
        torch.cuda.synchronize()

        def worker(i, n):
            for _ in range(n):
                one_stack(sess[i], frames[i], outs[i])

        per = steps // inflight
        t0 = time.perf_counter()
        th = [threading.Thread(target=worker, args=(i, per)) for i in range(inflight)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        dt = time.perf_counter() - t0
        ms = dt / (per * inflight) * 1e3
        results[inflight] = ms
        print(f"inflight={inflight}: {ms:.2f} ms per stack, {N / ms * 1e3:.0f} frames/s", flush=True)
        ref = outs[0].numpy().reshape(N, PLANE)
        for i in range(1, inflight):
            assert np.array_equal(outs[i].numpy().reshape(N, PLANE), ref), "sessions disagree"
        for s in sess:
            s.close()
        del frames, outs
    return results


if __name__ == "__main__":
    main()

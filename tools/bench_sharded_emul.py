"""Per-rank device time of the sharded pass, emulated on one GPU (G virtual ranks).

    python tools/bench_sharded_emul.py [G ...]

Each virtual rank runs its real work on cuda:0: the spatial step over its frame shard with
the fused corner-turn stores (into G local receive buffers instead of NVLink peers) and the
temporal step over its wave-vector slice. The max over ranks is the compute part of one
sharded step at G GPUs; the NVLink time of the stores (8 n_r (Q - Q_r) bytes per rank) is
estimated beside it at 900 GB/s per direction. C2 workload (512 x 512 x 1024).
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2012_05695_b200 import ddm, sharded  # noqa: E402

W, H, N = 512, 512, 1024


def emulate(G, reps=5):
    Q = H * (W // 2 + 1)
    plan = sharded.plan_shards(Q, N, G)
    st = ddm.generate(W, H, N, particles=100, diffusion=0.5, seed=7)
    frames = torch.from_numpy(st.view(np.int16)).cuda()
    ops = sharded.DeviceOps(W, H, "f32", device=0, timing=False)
    q_max = max(plan.q_of(d) for d in range(G))
    recvs = [torch.empty(2 * q_max * N, dtype=torch.float32, device="cuda") for _ in range(G)]
    outs = [torch.empty(N * max(plan.q_of(d), 1), dtype=torch.float32, device="cuda") for d in range(G)]
    stream = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    spatial, temporal = [], []
    for r in range(G):
        dest = [recvs[d].data_ptr() + plan.q_of(d) * plan.frame_begin[r] * 8 for d in range(G)]
        fr = frames[plan.frame_begin[r]: plan.frame_begin[r + 1]]
        for _ in range(2):
            ops.spatial_p2p(fr, plan.frames_of(r), plan.q_begin, dest)
        torch.cuda.synchronize()
        ev[0].record(stream)
        for _ in range(reps):
            ops.spatial_p2p(fr, plan.frames_of(r), plan.q_begin, dest)
        ev[1].record(stream)
        torch.cuda.synchronize()
        spatial.append(ev[0].elapsed_time(ev[1]) / reps)
    segs = [plan.frames_of(s) for s in range(G)]
    for d in range(G):
        q_d = plan.q_of(d)
        for _ in range(2):
            ops.temporal(recvs[d], q_d, segs, outs[d], q_d)
        torch.cuda.synchronize()
        ev[0].record(stream)
        for _ in range(reps):
            ops.temporal(recvs[d], q_d, segs, outs[d], q_d)
        ev[1].record(stream)
        torch.cuda.synchronize()
        temporal.append(ev[0].elapsed_time(ev[1]) / reps)
    sent = [8 * plan.frames_of(r) * (Q - plan.q_of(r)) for r in range(G)]
    nvlink_ms = max(sent) / 900e9 * 1e3
    step = max(spatial) + max(temporal)
    return {"G": G, "spatial_ms_max": max(spatial), "temporal_ms_max": max(temporal),
            "compute_step_ms": step, "frames_per_s_at_G": N / step * 1e3,
            "nvlink_bytes_per_rank": max(sent), "nvlink_ms_at_900GBps": nvlink_ms}


if __name__ == "__main__":
    for g in [int(x) for x in sys.argv[1:]] or [1, 2, 4, 8]:
        print(json.dumps(emulate(g)), flush=True)

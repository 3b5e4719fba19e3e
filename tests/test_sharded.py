"""Sharded WITH_FT: plan, corner-turn exchange, assembly.

CPU (`-m "not gpu"`): the shard plan through the C-ABI (host-only), and the whole sharded
pass at world size 2 and 3 under `gloo` with the numpy oracle standing in for the kernels —
the plan, the all-to-all block layout, the segment order the temporal step reads and the
assembly must reproduce the single-process oracle map exactly.

GPU (`-m gpu`): the device steps through the C-ABI with G virtual ranks on one GPU (the
exchange done as the same block copies the all-to-all performs) against the oracle and
against the unsharded device run, bitwise.
"""
import os
import socket

import numpy as np
import pytest

from oracle import ddm_oracle as O
from paper_2012_05695_b200 import ddm, sharded


# --------------------------------------------------------------------------- plan (host)

@pytest.mark.parametrize("q,n,g", [(131584, 1024, 2), (131584, 1024, 8), (2112, 128, 3),
                                   (125500, 1000, 8), (10, 7, 3), (5, 9, 4), (1, 2, 2)])
def test_plan_covers_and_aligns(q, n, g):
    p = sharded.plan_shards(q, n, g)
    assert p.frame_begin[0] == 0 and p.frame_begin[-1] == n
    assert p.q_begin[0] == 0 and p.q_begin[-1] == q
    fr = [p.frames_of(r) for r in range(g)]
    assert min(fr) >= 1 and max(fr) - min(fr) <= 2
    if n // 2 >= g:  # whole pairs: every segment but an odd tail is even
        assert all(f % 2 == 0 for f in fr[:-1])
        assert fr[-1] % 2 == n % 2
    # wave-vector slices are the reference GroupPlan with capacity ceil(Q / g)
    K = -(-q // g)
    assert list(p.q_begin) == [min(q, r * K) for r in range(g + 1)]
    assert sum(p.send_counts(0)) == q * fr[0]
    for r in range(g):
        assert sum(p.recv_counts(r)) == p.q_of(r) * n
        # what r sends to d is what d receives from r
        for d in range(g):
            assert p.send_counts(r)[d] == p.recv_counts(d)[r]


def test_plan_errors():
    with pytest.raises(ddm.InputError):
        sharded.plan_shards(100, 3, 4)      # fewer frames than ranks
    with pytest.raises(ddm.InputError):
        sharded.plan_shards(100, 64, 9)     # more than one node's 8 GPUs
    with pytest.raises(ddm.InputError):
        sharded.plan_shards(0, 64, 2)


def test_assemble_rejects_bad_partials():
    p = sharded.plan_shards(10, 8, 2)
    with pytest.raises(ddm.InputError):
        sharded.assemble(p, [np.zeros((8, 5)), np.zeros((8, 4))])


# --------------------------------------------------------------------------- gloo, CPU

class OracleOps:
    """Test checker standing in for the device kernels: the same buffers and layouts
    (send [Q][n_r], receive [source][Q_d][n_s]) filled by the numpy oracle."""

    def __init__(self, precision):
        self.precision = precision

    def spatial(self, frames_local, n_local, send):
        sp = O.spectra(frames_local.numpy(), self.precision).reshape(n_local, -1)
        qmaj = np.ascontiguousarray(sp.T)  # [Q][n_r]
        send.copy_(__import__("torch").from_numpy(qmaj.view(qmaj.real.dtype).reshape(-1)))

    def temporal(self, recv, q_count, seg_frames, out, out_stride, lags=None, out_f64=False):
        cdt = np.complex64 if self.precision == "f32" else np.complex128
        flat = recv.numpy().view(cdt)
        parts, base = [], 0
        for n_s in seg_frames:
            parts.append(flat[base: base + q_count * n_s].reshape(q_count, n_s))
            base += q_count * n_s
        seq = np.concatenate(parts, axis=1)
        d = O.with_ft(seq, self.precision)
        lag_list = O.normalize_lags(lags, seq.shape[1])
        vals = d[:, lag_list].T
        vals[np.asarray(lag_list) == 0] = 0.0
        o = out.numpy()
        for li in range(len(lag_list)):
            o[li * out_stride: li * out_stride + q_count] = vals[li]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, W, H, N, precision, lags, result_path):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        stack = O.random_stack(W, H, N, seed=5150)
        plan = sharded.plan_shards(H * (W // 2 + 1), N, world)
        local = torch.from_numpy(stack[plan.frame_begin[rank]: plan.frame_begin[rank + 1]].copy())
        run = sharded.ShardedRun(plan, rank, W, H, OracleOps(precision), precision=precision,
                                 lags=lags, out_f64=True)
        part = run.step(local)
        parts = sharded.gather_partials(plan, part, rank)
        if rank == 0:
            np.save(result_path, sharded.assemble(plan, parts))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,W,H,N,precision,lags", [
    (2, 16, 12, 20, "f64", None),
    (3, 10, 8, 17, "f64", [0, 1, 3, 16]),   # odd N: odd tail segment
    (2, 32, 32, 64, "f32", None),
    (4, 12, 10, 23, "f64", [0, 2, 22]),     # four ranks, odd N, uneven wave-vector slices
])
def test_gloo_sharded_matches_single_process(tmp_path, world, W, H, N, precision, lags):
    import torch.multiprocessing as mp
    out = tmp_path / "map.npy"
    mp.start_processes(_gloo_worker, args=(world, _free_port(), W, H, N, precision, lags, str(out)),
                       nprocs=world, join=True, start_method="spawn")
    got = np.load(out)
    stack = O.random_stack(W, H, N, seed=5150)
    ref = O.run_with_ft(stack, precision, lags=lags).reshape(got.shape)
    np.testing.assert_array_equal(got, ref)


# --------------------------------------------------------------------------- GPU

def _virtual_ranks(stack, G, precision="f32", lags=None, out_f64=True, exchange="copy"):
    """The sharded pass with G virtual ranks on cuda:0: per-rank spatial shards, the
    all-to-all as block copies ("copy") or the fused column-pass stores into every rank's
    receive buffer ("p2p", the NVLink path with local pointers), per-rank temporal over the
    segments; returns the map."""
    if exchange == "p2p":
        return _virtual_ranks_p2p(stack, G, lags, out_f64)
    import torch
    n, H, W = stack.shape
    Q = H * (W // 2 + 1)
    plan = sharded.plan_shards(Q, n, G)
    ops = sharded.DeviceOps(W, H, precision, device=0)
    real = torch.float32 if precision == "f32" else torch.float64
    frames = torch.from_numpy(stack.view(np.int16)).cuda()
    sends = []
    for r in range(G):
        send = torch.empty(2 * Q * plan.frames_of(r), dtype=real, device="cuda")
        ops.spatial(frames[plan.frame_begin[r]: plan.frame_begin[r + 1]], plan.frames_of(r), send)
        sends.append(send)
    parts = []
    n_lags = n if lags is None else len(lags)
    for d in range(G):
        # receive buffer of rank d: [source s][Q_d][n_s]
        chunks = [sends[s][2 * plan.q_begin[d] * plan.frames_of(s): 2 * plan.q_begin[d + 1] * plan.frames_of(s)]
                  for s in range(G)]
        recv = torch.cat(chunks)
        q_d = plan.q_of(d)
        out = torch.empty(n_lags * q_d, dtype=torch.float64 if out_f64 else torch.float32, device="cuda")
        ops.temporal(recv, q_d, [plan.frames_of(s) for s in range(G)], out, q_d, lags=lags,
                     out_f64=out_f64)
        parts.append(out.view(n_lags, q_d).cpu().numpy())
    torch.cuda.synchronize()
    return sharded.assemble(plan, parts).reshape(n_lags, H, W // 2 + 1)


def _virtual_ranks_p2p(stack, G, lags=None, out_f64=True):
    import torch
    n, H, W = stack.shape
    Q = H * (W // 2 + 1)
    plan = sharded.plan_shards(Q, n, G)
    ops = sharded.DeviceOps(W, H, "f32", device=0)
    frames = torch.from_numpy(stack.view(np.int16)).cuda()
    q_max = max(plan.q_of(d) for d in range(G))
    recvs = [torch.full((2 * q_max * n,), float("nan"), dtype=torch.float32, device="cuda")
             for _ in range(G)]
    for r in range(G):
        dest = [recvs[d].data_ptr() + plan.q_of(d) * plan.frame_begin[r] * 8 for d in range(G)]
        ops.spatial_p2p(frames[plan.frame_begin[r]: plan.frame_begin[r + 1]], plan.frames_of(r),
                        plan.q_begin, dest)
    parts = []
    n_lags = n if lags is None else len(lags)
    for d in range(G):
        q_d = plan.q_of(d)
        out = torch.empty(n_lags * q_d, dtype=torch.float64 if out_f64 else torch.float32, device="cuda")
        ops.temporal(recvs[d], q_d, [plan.frames_of(s) for s in range(G)], out, q_d, lags=lags,
                     out_f64=out_f64)
        parts.append(out.view(n_lags, q_d).cpu().numpy())
    torch.cuda.synchronize()
    return sharded.assemble(plan, parts).reshape(n_lags, H, W // 2 + 1)


@pytest.mark.gpu
@pytest.mark.parametrize("G", [2, 8])
def test_gpu_fused_p2p_corner_turn(G):
    """The fused corner turn (column pass storing into the owners' receive buffers) with G
    virtual ranks: bitwise equal to the unsharded run on the C2 geometry."""
    st = ddm.generate(512, 512, 1024, particles=100, diffusion=0.5, seed=7)
    got = _virtual_ranks(st, G, exchange="p2p")
    ref = ddm.run(st, ddm.RunConfig(precision="f32", memory_bytes=1 << 40)).values
    np.testing.assert_array_equal(got, ref)


@pytest.mark.gpu
def test_gpu_fused_p2p_small_and_errors():
    st = O.random_stack(128, 64, 96, seed=3)
    got = _virtual_ranks(st, 3, exchange="p2p")
    assert O.relative_l2(got, O.run_with_ft(st, "f32")) <= 1e-4
    # non power-of-two frames have no register-resident column pass: refused, not faked
    import torch
    ops = sharded.DeviceOps(30, 20, "f32", device=0)
    fr = torch.zeros(30 * 20 * 4, dtype=torch.int16, device="cuda")
    buf = torch.zeros(2 * 20 * 16 * 4, dtype=torch.float32, device="cuda")
    with pytest.raises(ddm.InputError):
        ops.spatial_p2p(fr, 4, [0, 20 * 16], [buf.data_ptr()])


@pytest.mark.gpu
@pytest.mark.parametrize("G", [1, 2, 3, 8])
def test_gpu_virtual_ranks_c2_geometry(G):
    """512x512 frames (the register-resident engines), N=1024 as C2 but fewer... full N."""
    st = ddm.generate(512, 512, 1024, particles=100, diffusion=0.5, seed=7)
    got = _virtual_ranks(st, G)
    ref = ddm.run(st, ddm.RunConfig(precision="f32", memory_bytes=1 << 40)).values
    # the sharded path is the same arithmetic per sequence: bitwise equal to the single run
    np.testing.assert_array_equal(got, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("W,H,N,G,precision,lags", [
    (64, 64, 128, 2, "f32", None),
    (64, 48, 100, 3, "f64", None),          # generic engines + repack path
    (30, 20, 33, 4, "f32", [0, 1, 5, 32]),  # odd N, odd tail segment, lag subset
    (32, 32, 1500, 3, "f32", None),         # long-sequence engine reading segments (R = 4)
    (16, 16, 2100, 8, "f32", [0, 3, 2099]), # long-sequence engine, R = 8
])
def test_gpu_virtual_ranks_vs_oracle(W, H, N, G, precision, lags):
    st = O.random_stack(W, H, N, seed=77)
    got = _virtual_ranks(st, G, precision, lags)
    ref = O.run_with_ft(st, precision, lags=lags)
    tol = 1e-4 if precision == "f32" else 1e-10
    assert O.relative_l2(got, ref) <= tol



# --------------------------------------------------------------------------- sharded ring average

def _ring_worker(rank, world, port, result_path):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # rank r's slice of a 20 x 17 plane map (3 lags): its ring sums and counts, by the
        # oracle's ring assignment; ring_average must equal the whole-map ring means
        W, H, L = 32, 20, 3
        Q = H * (W // 2 + 1)
        vals = np.random.default_rng(3).uniform(0, 5, size=(L, Q))
        plan = sharded.plan_shards(Q, 8 * world, world)
        b, e = plan.q_begin[rank], plan.q_begin[rank + 1]
        hc = W // 2 + 1
        ks = np.arange(Q)
        bins = np.floor(O.q_magnitude(ks // hc, ks % hc, H) + 0.5).astype(np.int64)
        nb = int(bins.max()) + 1
        sums = np.zeros((L, nb))
        for li in range(L):
            sums[li] = np.bincount(bins[b:e], weights=vals[li, b:e], minlength=nb)
        counts = np.bincount(bins[b:e], minlength=nb)
        means, cnt = sharded.ring_average(torch.from_numpy(sums), counts)
        if rank == 0:
            np.save(result_path, {"means": means.numpy(), "counts": cnt, "vals": vals}, allow_pickle=True)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_ring_average_matches_whole_map(tmp_path, world):
    import torch.multiprocessing as mp
    out = tmp_path / "ring.npy"
    mp.spawn(_ring_worker, args=(world, _free_port(), str(out)), nprocs=world, join=True)
    r = np.load(out, allow_pickle=True).item()
    means, counts = O.azimuthal_average(r["vals"].reshape(3, 20, 17), 32, 20)
    assert np.array_equal(r["counts"], counts)
    assert np.allclose(r["means"], means, rtol=1e-12, atol=0)


@pytest.mark.gpu
@pytest.mark.parametrize("G", [1, 2, 3])
def test_gpu_sharded_ring_sums_match_azimuthal(G):
    """Per-rank ring sums (ddm_b200_ring_sums_device) over the sharded temporal outputs,
    added in rank order, equal the ring means of the assembled map (`analysis.cpp:61-97`)."""
    import torch
    from paper_2012_05695_b200 import ddm
    W, H, N = 64, 48, 96
    st = ddm.generate(W, H, N, particles=30, seed=12)
    Q = H * (W // 2 + 1)
    plan = sharded.plan_shards(Q, N, G)
    ops = sharded.DeviceOps(W, H, "f32", device=0)
    frames = torch.from_numpy(st.view(np.int16)).cuda()
    sends = []
    for r in range(G):
        send = torch.empty(2 * Q * plan.frames_of(r), dtype=torch.float32, device="cuda")
        ops.spatial(frames[plan.frame_begin[r]: plan.frame_begin[r + 1]], plan.frames_of(r), send)
        sends.append(send)
    sums, counts, parts = [], [], []
    for d in range(G):
        chunks = [sends[s][2 * plan.q_begin[d] * plan.frames_of(s): 2 * plan.q_begin[d + 1] * plan.frames_of(s)]
                  for s in range(G)]
        q_d = plan.q_of(d)
        out = torch.empty(N * q_d, dtype=torch.float32, device="cuda")
        ops.temporal(torch.cat(chunks), q_d, [plan.frames_of(s) for s in range(G)], out, q_d)
        s_d, c_d = ops.ring_sums(out, plan.q_begin[d], q_d, q_d, N)
        sums.append(s_d)
        counts.append(c_d)
        parts.append(out.view(N, q_d).cpu().numpy().astype(np.float64))
    means, cnt = sharded.combine_ring_sums(sums, counts)
    full = sharded.assemble(plan, parts)
    ref_means, ref_counts = O.azimuthal_average(full.reshape(N, H, W // 2 + 1), W, H)
    assert np.array_equal(cnt, ref_counts)
    got = means.cpu().numpy()
    assert np.abs(got - ref_means).max() <= 1e-12 * np.abs(ref_means).max()

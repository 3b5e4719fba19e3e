"""Sharded WITH_FT over several GPUs of one node.

One process per GPU. The reference is a single process whose out-of-core path slices the
wave vectors into contiguous groups (`plan_with_ft`, `scheduler.cpp:365-384`) and loops all
frames per group (`scheduler.cpp:89-171`). Here the two loops are split across ranks:

  step 1  rank r transforms its frame shard [f_r, f_{r+1}) for every wave vector
          (`ddm_b200_spatial_shard_device`): send buffer [Q][n_r], q-major, so the rows
          [q_d, q_{d+1}) are the block for rank d;
  corner  all-to-all (NCCL over NVLink via torch.distributed): rank d receives
  turn    [source s][Q_d][n_s], the full sequences of its wave-vector slice in segments;
  step 2  rank d runs the fused temporal engine over its slice, reading the segments in
          place (`ddm_b200_temporal_segments_device`): lag-major [lags][Q_d], exactly the
          reference's PartialResult of group d (`archive.hpp:48-61`).

The map never crosses ranks: each rank keeps its partial in HBM (`assemble` gathers them for
tests and host output, which is the reference's merge_partials).

The compute steps are an injected `ops` object so the plan / exchange / assembly logic runs
under `gloo` on CPU in the tests with a checker in place of the kernels; the product path is
`DeviceOps`, which calls the C-ABI and has no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import ddm


@dataclass(frozen=True)
class ShardPlan:
    """ddm::ShardPlan (include/ddm/scheduler.hpp): offsets with ranks + 1 entries each."""
    ranks: int
    frames: int
    q_count: int
    frame_begin: tuple
    q_begin: tuple

    def frames_of(self, r: int) -> int:
        return self.frame_begin[r + 1] - self.frame_begin[r]

    def q_of(self, r: int) -> int:
        return self.q_begin[r + 1] - self.q_begin[r]

    def send_counts(self, r: int) -> List[int]:
        """complex values rank r sends to each destination (its frames x their slice)."""
        return [self.q_of(d) * self.frames_of(r) for d in range(self.ranks)]

    def recv_counts(self, r: int) -> List[int]:
        """complex values rank r receives from each source (its slice x their frames)."""
        return [self.q_of(r) * self.frames_of(s) for s in range(self.ranks)]


def plan_shards(q_count: int, frames: int, ranks: int) -> ShardPlan:
    """ddm::plan_shards through the C-ABI (host-only; no device needed)."""
    fb = np.zeros(ranks + 1, dtype=np.int64)
    qb = np.zeros(ranks + 1, dtype=np.int64)
    ddm._check(ddm.lib().ddm_b200_shard_plan(C.c_int64(q_count), C.c_int64(frames), int(ranks),
                                             ddm._p(fb, C.c_int64), ddm._p(qb, C.c_int64)))
    return ShardPlan(int(ranks), int(frames), int(q_count), tuple(int(x) for x in fb),
                     tuple(int(x) for x in qb))


class DeviceOps:
    """The product compute steps: C-ABI kernels on the rank's GPU (torch tensors as HBM)."""

    def __init__(self, width: int, height: int, precision: str = "f32", device: int = 0,
                 pixel_bytes: int = 2, timing: bool = True):
        self.width, self.height = width, height
        self.timing = timing  # per-step device times (synchronises the host per step)
        self.precision = precision
        self.device = device
        self.pixel_bytes = pixel_bytes
        self.spatial_ms = 0.0
        self.temporal_ms = 0.0

    def _stream(self):
        import torch
        return torch.cuda.current_stream(self.device).cuda_stream

    def spatial(self, frames_local, n_local: int, send) -> None:
        """frames_local: device tensor of the shard's pixels; send: device tensor of
        Q * n_local complex values (real pairs)."""
        ms = C.c_double(0.0)
        ddm._check(ddm.lib().ddm_b200_spatial_shard_device(
            C.c_void_p(frames_local.data_ptr()), self.pixel_bytes, self.width, self.height,
            int(n_local), 0 if self.precision == "f32" else 1, C.c_void_p(send.data_ptr()),
            self.device, C.c_void_p(self._stream()), C.byref(ms) if self.timing else None))
        self.spatial_ms = ms.value

    def spatial_p2p(self, frames_local, n_local: int, q_begin: Sequence[int],
                    dest: Sequence[int]) -> None:
        """Step 1 fused with the corner turn: the column pass stores every wave vector of
        the shard straight into its owner's receive buffer (`dest[d]`, device pointers valid
        on this GPU: peer mappings over NVLink, already offset to this rank's segment)."""
        qb = np.ascontiguousarray(np.asarray(q_begin, dtype=np.int64))
        ptrs = (C.c_void_p * len(dest))(*[C.c_void_p(int(x)) for x in dest])
        ms = C.c_double(0.0)
        ddm._check(ddm.lib().ddm_b200_spatial_shard_p2p_device(
            C.c_void_p(frames_local.data_ptr()), self.pixel_bytes, self.width, self.height,
            int(n_local), 0 if self.precision == "f32" else 1, len(dest), ddm._p(qb, C.c_int64),
            ptrs, self.device, C.c_void_p(self._stream()), C.byref(ms) if self.timing else None))
        self.spatial_ms = ms.value

    def temporal(self, recv, q_count: int, seg_frames: Sequence[int], out, out_stride: int,
                 lags: Optional[Sequence[int]] = None, out_f64: bool = False) -> None:
        segs = np.ascontiguousarray(np.asarray(seg_frames, dtype=np.int64))
        lag_arr = np.ascontiguousarray(np.asarray(lags if lags is not None else [], dtype=np.int64))
        ms = C.c_double(0.0)
        ddm._check(ddm.lib().ddm_b200_temporal_segments_device(
            C.c_void_p(recv.data_ptr()), C.c_int64(q_count), len(segs), ddm._p(segs, C.c_int64),
            0 if self.precision == "f32" else 1,
            ddm._p(lag_arr, C.c_int64) if len(lag_arr) else None, C.c_int64(len(lag_arr)),
            C.c_void_p(out.data_ptr()), C.c_int64(out_stride), 1 if out_f64 else 0, self.device,
            C.c_void_p(self._stream()), C.byref(ms) if self.timing else None))
        self.temporal_ms = ms.value


    def ring_sums(self, out, q_begin: int, q_count: int, out_stride: int, n_lags: int,
                  out_f64: bool = False, q_max: Optional[float] = None):
        """Per-(lag, ring) sums of this rank's slice [q_begin, q_begin + q_count) of the map
        (device tensor [n_lags][out_stride]) -> (sums: device f64 tensor [n_lags, bins],
        counts: numpy int64 [bins]). Every rank gets the same bin count."""
        import torch
        nb = C.c_int64(0)
        args = (C.c_int64(q_begin), C.c_int64(q_count), C.c_int64(out_stride), C.c_int64(n_lags),
                self.width, self.height, 0 if q_max is None else 1, C.c_double(q_max or 0.0))
        ddm._check(ddm.lib().ddm_b200_ring_sums_device(
            C.c_void_p(out.data_ptr()), 1 if out_f64 else 0, *args, None, C.c_int64(0), None,
            C.byref(nb), self.device, C.c_void_p(self._stream())))
        sums = torch.empty(n_lags, nb.value, dtype=torch.float64, device=out.device)
        counts = np.zeros(max(nb.value, 1), dtype=np.int64)
        ddm._check(ddm.lib().ddm_b200_ring_sums_device(
            C.c_void_p(out.data_ptr()), 1 if out_f64 else 0, *args, C.c_void_p(sums.data_ptr()),
            C.c_int64(sums.numel()), ddm._p(counts, C.c_int64), C.byref(nb), self.device,
            C.c_void_p(self._stream())))
        return sums, counts[: nb.value]


def combine_ring_sums(sums: Sequence, counts: Sequence):
    """Ring means from the ranks' (sums, counts), added in rank order (deterministic):
    mean = sum / count, empty rings 0 (`analysis.cpp:61-97`). Works on torch tensors or numpy."""
    total = sums[0].clone() if hasattr(sums[0], "clone") else np.array(sums[0], dtype=np.float64)
    for t in sums[1:]:
        total += t
    cnt = np.asarray(counts[0], dtype=np.int64).copy()
    for c in counts[1:]:
        cnt += np.asarray(c, dtype=np.int64)
    if hasattr(total, "clone"):
        import torch
        ct = torch.as_tensor(cnt, device=total.device)
        means = torch.where(ct > 0, total / ct.clamp(min=1).to(total.dtype), torch.zeros_like(total))
    else:
        means = np.where(cnt > 0, total / np.maximum(cnt, 1), 0.0)
    return means, cnt


def ring_average(sums, counts, group=None):
    """Sharded ring average, step 2: gather every rank's [lags, bins] sums and
    ring counts (a few MB), add them in rank order and divide. Returns (means, counts) on
    every rank."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return combine_ring_sums([sums], [counts])
    world = dist.get_world_size(group)
    ct = torch.as_tensor(np.asarray(counts, dtype=np.int64), device=sums.device)
    s_all = [torch.empty_like(sums) for _ in range(world)]
    c_all = [torch.empty_like(ct) for _ in range(world)]
    dist.all_gather(s_all, sums.contiguous(), group=group)
    dist.all_gather(c_all, ct, group=group)
    return combine_ring_sums(s_all, [c.cpu().numpy() for c in c_all])


class ShardedRun:
    """One rank of a sharded WITH_FT run. Buffers are allocated once and reused per step.

    Scalars travel as real pairs: f32 runs exchange float32 tensors, f64 runs float64.
    """

    def __init__(self, plan: ShardPlan, rank: int, width: int, height: int, ops, *,
                 precision: str = "f32", device=None, group=None, lags=None,
                 out_f64: bool = False, exchange: str = "nccl"):
        import torch
        self.torch = torch
        self.plan, self.rank = plan, rank
        self.width, self.height = width, height
        if plan.q_count != height * (width // 2 + 1):
            raise ddm.InputError("plan q_count must be the half-plane size H*(W/2+1)")
        self.ops, self.group = ops, group
        self.precision = precision
        self.lags = None if lags is None else [int(x) for x in lags]
        self.n_lags = plan.frames if lags is None else len(self.lags)
        self.out_f64 = out_f64
        real = torch.float32 if precision == "f32" else torch.float64
        dev = torch.device("cpu") if device is None else torch.device(device)
        Q, n_r = plan.q_count, plan.frames_of(rank)
        if exchange not in ("nccl", "p2p"):
            raise ddm.InputError("exchange must be 'nccl' or 'p2p'")
        self.exchange_mode = exchange
        self.symm = None
        if exchange == "p2p":
            # receive buffers in symmetric memory: every rank maps every peer's buffer, the
            # column pass stores into them directly (equal sizes on all ranks)
            import torch.distributed._symmetric_memory as symm
            import torch.distributed as dist
            q_max = max(plan.q_of(r) for r in range(plan.ranks))
            self.recv = symm.empty(2 * q_max * plan.frames, dtype=real, device=dev)
            self.symm = symm.rendezvous(self.recv, group if group is not None else dist.group.WORLD)
            csize = 8 if precision == "f32" else 16
            ptrs = list(self.symm.buffer_ptrs)
            # this rank's segment in rank d's buffer: [source][Q_d][n_s], sources before it
            self.dest = [int(ptrs[d]) + plan.q_of(d) * plan.frame_begin[rank] * csize
                         for d in range(plan.ranks)]
            self.send = None
        else:
            self.send = torch.empty(2 * Q * n_r, dtype=real, device=dev)
            # one rank: the send buffer already is the single-source receive buffer
            self.recv = (self.send if plan.ranks == 1 else
                         torch.empty(2 * plan.q_of(rank) * plan.frames, dtype=real, device=dev))
        self.out = torch.empty(self.n_lags * max(plan.q_of(rank), 1),
                               dtype=torch.float64 if out_f64 else torch.float32, device=dev)
        self.send_splits = [2 * c for c in plan.send_counts(rank)]
        self.recv_splits = [2 * c for c in plan.recv_counts(rank)]
        self.seg_frames = [plan.frames_of(s) for s in range(plan.ranks)]

    def spatial(self, frames_local) -> None:
        """Step 1 (with the stores of the fused corner turn in p2p mode)."""
        n_r = self.plan.frames_of(self.rank)
        if self.symm is not None:
            self.symm.barrier(channel=0)   # every peer has consumed its previous receive buffer
            self.ops.spatial_p2p(frames_local, n_r, self.plan.q_begin, self.dest)
        else:
            self.ops.spatial(frames_local, n_r, self.send)

    def exchange(self) -> None:
        """The corner turn: every rank's [Q_d][n_r] block to rank d (p2p: the blocks are
        already in place; wait until every rank's stores have landed)."""
        if self.symm is not None:
            self.symm.barrier(channel=1)
            return
        if self.plan.ranks == 1:
            return
        import torch.distributed as dist
        dist.all_to_all_single(self.recv, self.send, self.recv_splits, self.send_splits,
                               group=self.group)

    def step(self, frames_local):
        """Whole sharded pass for this rank; returns the rank's lag-major partial
        [n_lags][Q_r] (a view of `self.out`)."""
        self.spatial(frames_local)
        self.exchange()
        q_r = self.plan.q_of(self.rank)
        if q_r > 0:
            self.ops.temporal(self.recv, q_r, self.seg_frames, self.out, q_r, lags=self.lags,
                              out_f64=self.out_f64)
        return self.out[: self.n_lags * q_r].view(self.n_lags, q_r)


def assemble(plan: ShardPlan, partials: Sequence[np.ndarray]) -> np.ndarray:
    """merge_partials over the ranks' outputs (`scheduler.cpp:485-542` with identity flat
    positions): [n_lags][Q] from the per-rank [n_lags][Q_r] blocks."""
    blocks = [np.asarray(p) for p in partials]
    n_lags = blocks[0].shape[0]
    out = np.zeros((n_lags, plan.q_count), dtype=np.float64)
    for r, b in enumerate(blocks):
        if b.shape != (n_lags, plan.q_of(r)):
            raise ddm.InputError(f"partial of rank {r} has shape {b.shape}, "
                                 f"expected {(n_lags, plan.q_of(r))}")
        out[:, plan.q_begin[r]:plan.q_begin[r + 1]] = b
    return out


def gather_partials(plan: ShardPlan, partial, rank: int, group=None):
    """Collect every rank's partial on rank 0 (host numpy), None elsewhere."""
    import torch
    import torch.distributed as dist
    if plan.ranks == 1:
        return [partial.detach().cpu().numpy()]
    n_lags = partial.shape[0]
    width = max(plan.q_of(r) for r in range(plan.ranks))
    padded = torch.zeros(n_lags, width, dtype=partial.dtype, device=partial.device)
    padded[:, : partial.shape[1]] = partial
    bufs = [torch.zeros_like(padded) for _ in range(plan.ranks)] if rank == 0 else None
    dist.gather(padded, bufs, dst=0, group=group)
    if rank != 0:
        return None
    return [b[:, : plan.q_of(r)].cpu().numpy() for r, b in enumerate(bufs)]

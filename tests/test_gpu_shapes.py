"""GPU parity at the BASELINE shapes the register engines specialise on.

BASELINE configs[2] (C3: 1024^2 x 2048 with q-ring averaging) and configs[3] (C4: 2048^2 x
4096, here on one B200) select kernels no smaller shape reaches: rows2<512>/<1024>,
cols2<1024>/<2048>, the long-sequence engine long2<4>/<8> and its multi-chunk lag transpose
(q0 > 0 offsets). Each case runs through the device C-ABI (`ddm_b200_run_device`, frames and
map in HBM), asserts which kernels ran (`ddm_b200_last_engines`), and compares a subset of wave
vectors with the oracle's `with_ft` (`oracle/ddm_oracle.py`, restating `temporal.cpp:77-129`)
in f64 on spectra from an independent f64 FFT (torch.fft on the device, test-only checker).
Tolerance: the north-star f32 bound, relative L2 <= 1e-4 (`BASELINE.json`).

Frames are per-pixel random walks around a random background (so d(q, m) grows with m and
the small-lag entries cancel as in real DDM data), generated on the device.
"""
import numpy as np
import pytest

from oracle import ddm_oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

F32_L2 = 1e-4


@pytest.fixture(scope="module")
def env():
    torch = pytest.importorskip("torch")
    from paper_2012_05695_b200 import ddm as D
    if D.device_count() < 1 or not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch, D


def walk_frames(torch, W, H, N, seed):
    """[N, H, W] u16 frames (held as int16: values stay below 2^15) on cuda:0."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    cur = torch.randint(500, 3000, (H, W), generator=g, device="cuda", dtype=torch.int32)
    out = torch.empty((N, H, W), dtype=torch.int16, device="cuda")
    for n in range(N):
        cur += torch.randint(-8, 9, (H, W), generator=g, device="cuda", dtype=torch.int32)
        cur.clamp_(0, 32767)
        out[n] = cur.to(torch.int16)
    return out


def ref_spectra(torch, frames, idx, chunk_bytes=1 << 30):
    """f64 half-plane spectra of every frame at the flat wave vectors idx: [N, K] complex128."""
    N, H, W = frames.shape
    it = torch.as_tensor(idx, device="cuda")
    step = max(1, chunk_bytes // (H * W * 16))
    out = []
    for f0 in range(0, N, step):
        x = frames[f0:f0 + step].to(torch.int32).to(torch.float64)
        X = torch.fft.rfft2(x).reshape(x.shape[0], -1)
        out.append(X.index_select(1, it).cpu())
        del x, X
    torch.cuda.empty_cache()
    return torch.cat(out).numpy()


def pick(Q, k, seed):
    """k wave vectors: the plane's first and last ones plus a random spread."""
    r = np.random.default_rng(seed)
    idx = np.unique(np.concatenate([[0, 1, Q - 2, Q - 1], r.choice(Q, k, replace=False)]))
    return idx.astype(np.int64)


def run_case(torch, D, W, H, N, seed, k=512, expect=()):
    Q = H * (W // 2 + 1)
    frames = walk_frames(torch, W, H, N, seed)
    idx = pick(Q, k, seed)
    spec = ref_spectra(torch, frames, idx)
    ref = O.with_ft(np.ascontiguousarray(spec.T), "f64").T
    ref[0] = 0.0
    out = torch.empty((N, Q), dtype=torch.float32, device="cuda")
    D.run_device(frames.data_ptr(), 2, W, H, N, out.data_ptr(), "f32")
    eng = D.last_engines()
    for e in expect:
        assert e in eng, (e, eng)
    got = out.index_select(1, torch.as_tensor(idx, device="cuda")).cpu().numpy().astype(np.float64)
    # whole-map properties at full size (lag chunks, no map-sized temporaries): d(0) == 0
    # exactly, finite, the validate() floor (`archive.cpp:44-58`)
    assert bool(torch.all(out[0] == 0))
    peak, low = 0.0, 0.0
    for l0 in range(0, N, 64):
        blk = out[l0:l0 + 64]
        assert bool(torch.isfinite(blk).all())
        peak = max(peak, float(blk.max()))
        low = min(low, float(blk.min()))
    assert low >= -1e-4 * max(peak, 1.0)
    err = O.relative_l2(got, ref)
    print(f"{W}x{H}x{N}: relative L2 {err:.3e} over {len(idx)} wave vectors [{eng}]")
    assert err <= F32_L2, (W, H, N, err, eng)
    return frames, out, err


@pytest.mark.parametrize("W,H,N,expect", [
    (128, 2048, 600, ("cols2<2048>", "warp<1024>")),
    (1024, 1024, 600, ("rows2<512>", "cols2<1024>", "warp<1024>")),
    (1024, 256, 2048, ("rows2<512>", "long2<4>", "chunks=2")),      # Q = 131328 > 131072
    (2048, 128, 4096, ("rows2<1024>", "long2<8>", "chunks=3")),     # Q = 131200 > 2 x 65536
])
def test_engine_shapes_vs_oracle(env, W, H, N, expect):
    torch, D = env
    frames, out, err = run_case(torch, D, W, H, N, seed=W + H + N, expect=expect)
    del frames, out
    torch.cuda.empty_cache()


def test_c3_map_and_rings(env):
    """BASELINE configs[2]: 1024^2 x 2048. Map subset vs the oracle, then the fused ring
    average (no map) against the map's own ring average (`analysis.cpp:61-97`)."""
    torch, D = env
    W = H = 1024
    N = 2048
    frames, out, err = run_case(torch, D, W, H, N, seed=3,
                                expect=("rows2<512>", "cols2<1024>", "long2<4>", "chunks=5"))
    # ring average of the device map, lag by lag in f64, bins from the oracle's geometry
    flat = O.cutoff_set(W, H)
    hc = O.half_cols(W)
    bins = np.floor(O.q_magnitude(flat // hc, flat % hc, H) + 0.5).astype(np.int64)
    nb = int(bins.max()) + 1
    counts = np.bincount(bins, minlength=nb)
    b_t = torch.as_tensor(bins, device="cuda")
    sums = torch.zeros((N, nb), dtype=torch.float64, device="cuda")
    for l0 in range(0, N, 256):
        sums[l0:l0 + 256].index_add_(1, b_t, out[l0:l0 + 256].to(torch.float64))
    map_means = (sums / torch.as_tensor(counts, device="cuda").clamp(min=1)).cpu().numpy()
    del out, sums
    torch.cuda.empty_cache()
    means = torch.zeros((N, nb), dtype=torch.float64, device="cuda")
    nbins, _, _, fused = D.run_azimuthal_device(frames.data_ptr(), 2, W, H, N, means.data_ptr(), nb)
    assert fused and nbins == nb
    assert "long2<4>" in D.last_engines() and ":ring" in D.last_engines()
    m = means.cpu().numpy()
    assert np.all(m[0] == 0.0)
    assert O.relative_l2(m, map_means) <= 1e-5
    del frames, means
    torch.cuda.empty_cache()


def test_c4_one_gpu(env):
    """BASELINE configs[3] geometry on one B200: 2048^2 x 4096 (frames 34 GB, map 34 GB,
    spectra 69 GB resident)."""
    torch, D = env
    free, _ = torch.cuda.mem_get_info()
    if free < 150e9:
        pytest.skip(f"needs ~145 GB of free HBM, {free / 1e9:.0f} GB free")
    frames, out, err = run_case(torch, D, 2048, 2048, 4096, seed=4, k=384,
                                expect=("rows2<1024>", "cols2<2048>", "long2<8>", "chunks=33"))
    del frames, out
    torch.cuda.empty_cache()


def test_c2_full_map_vs_oracle(env):
    """BASELINE configs[1] (512^2 x 1024, f32), every one of the 131,584 x 1,024 map entries
    against the f64 oracle through the reference-facing host call (`ddm::run`)."""
    torch, D = env
    st = D.generate(512, 512, 1024, particles=100, diffusion=0.5, seed=7)
    a = D.run(st, D.RunConfig(precision="f32", memory_bytes=1 << 40))
    eng = D.last_engines()
    assert "rows2<256>" in eng and "cols2<512>" in eng and "warp<1024>" in eng, eng
    got = a.values.reshape(1024, -1)
    sp = O.spectra(st, "f64").reshape(1024, -1)
    num = den = 0.0
    for q0 in range(0, sp.shape[1], 8192):
        ref = O.with_ft(np.ascontiguousarray(sp[:, q0:q0 + 8192].T), "f64").T
        ref[0] = 0.0
        num += float(np.sum((got[:, q0:q0 + 8192] - ref) ** 2))
        den += float(np.sum(ref ** 2))
    assert np.sqrt(num / den) <= F32_L2

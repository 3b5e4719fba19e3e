"""ORACLE / TEST INFRASTRUCTURE ONLY — numpy restatement of the reference WITH_FT path.

This module is the CPU checker for the CUDA product path.  It restates, in vectorised
numpy, the reference's FFT-in-time structure function exactly as the C++ computes it:
  * spatial step: unnormalised r2c 2D over (rows=H, cols=W) in the working precision
    (`proj/core/src/fft.cpp:34-37,86-87,128-132`; conversion `scheduler.cpp:115-119`);
  * per wave vector: mean in complex128, cast to the working precision S, subtract in S
    (`temporal.cpp:82-92`); averages term with f64 power (`temporal.cpp:19-42`, prefix-sum
    form); zero-pad to pad_length, forward FFT, |X|^2 in S, inverse FFT, scale 1/N2 in f64,
    real part of the first N (`temporal.cpp:48-75`); combine in f64 (`temporal.cpp:114-129`);
  * d(0) := 0 and only the requested lags (`scheduler.cpp:155-161`); wave vectors outside
    the cutoff stay 0 (`scheduler.cpp:432-444`, `merge_partials` `:485-542`).
It is pinned against the reference itself (oracle/_ref, tests/golden/) and the reference's
known-answer tests (tests/test_oracle.py).  Only tests/, bench.py's cpu_baseline leg and
__graft_entry__.smoke() may import it.
"""
from __future__ import annotations

import math

import numpy as np

_REAL = {"f32": np.float32, "f64": np.float64}
_CPLX = {"f32": np.complex64, "f64": np.complex128}


def pad_length(frames: int) -> int:
    """`temporal.cpp:10-17`: 2^(ceil(log2 N) + 1)."""
    if frames < 1:
        raise ValueError("pad_length: sequence must have at least one frame")
    n2 = 1
    while n2 < frames:
        n2 <<= 1
    return n2 << 1


def half_cols(width: int) -> int:
    """`spectrum.hpp:16`."""
    return width // 2 + 1


def q_magnitude(row, col, height):
    """`spectrum.hpp:20-24` (vectorised)."""
    row = np.asarray(row)
    q_row = np.where(row <= height // 2, row, row - height).astype(np.float64)
    col = np.asarray(col, dtype=np.float64)
    return np.sqrt(q_row * q_row + col * col)


def cutoff_set(width: int, height: int, q_max=None) -> np.ndarray:
    """`spectrum.cpp:65-84`: row-major flat indices of the retained half-plane positions."""
    if width < 1 or height < 1:
        raise ValueError("cutoff_set: dimensions must be positive")
    if q_max is not None and q_max < 0:
        raise ValueError("cutoff_set: q_max must be non-negative")
    hc = half_cols(width)
    flat = np.arange(height * hc, dtype=np.int64)
    if q_max is None:
        return flat
    keep = q_magnitude(flat // hc, flat % hc, height) <= q_max
    return flat[keep]


def plan_with_ft(q_count: int, frames: int, nbytes: int, precision: str = "f64"):
    """`scheduler.cpp:365-384`: capacity K and [begin, end) groups."""
    if frames < 1 or q_count < 1:
        raise ValueError("plan_with_ft: bad sizes")
    per = frames * (8 if precision == "f32" else 16)
    cap = nbytes // per if nbytes > 0 else 0
    if cap < 1:
        raise MemoryError("plan_with_ft: budget cannot hold one sequence")
    return cap, [(b, min(b + cap, q_count)) for b in range(0, q_count, cap)]


# --------------------------------------------------------------------------- temporal


def averages_term(seqs: np.ndarray) -> np.ndarray:
    """`temporal.cpp:19-42` for a batch [Q, N] (any complex dtype), in f64.

    d_a(m) = (sum_{n<N-m} p_n + sum_{n>=m} p_n) / (N-m), p_n = |s_n|^2 in f64.  The
    reference evaluates it by a backward recursion; prefix sums are the same quantity.
    """
    s = np.asarray(seqs)
    p = s.real.astype(np.float64) ** 2 + s.imag.astype(np.float64) ** 2
    n = p.shape[-1]
    c = np.concatenate([np.zeros(p.shape[:-1] + (1,)), np.cumsum(p, axis=-1)], axis=-1)
    m = np.arange(n)
    head = c[..., n - m]          # sum_{n < N-m}
    tail = c[..., n:n + 1] - c[..., m]  # sum_{n >= m}
    return (head + tail) / (n - m)


def correlation(seqs: np.ndarray, precision: str = "f64") -> np.ndarray:
    """`temporal.cpp:48-75`: Re of the linear autocorrelation via zero-padded FFT."""
    s = np.asarray(seqs, dtype=_CPLX[precision])
    n = s.shape[-1]
    n2 = pad_length(n)
    x = np.fft.fft(s, n=n2, axis=-1)          # zero-padded, sign -1 (`fft.cpp:157`)
    x = x.astype(_CPLX[precision], copy=False)
    pw = (x.real * x.real + x.imag * x.imag).astype(_REAL[precision])
    r = np.fft.ifft(pw.astype(_CPLX[precision]), axis=-1) * n2  # unnormalised backward
    r = r.astype(_CPLX[precision], copy=False)
    return r.real[..., :n].astype(np.float64) * (1.0 / n2)


def with_ft(seqs: np.ndarray, precision: str = "f64"):
    """`SequenceEngine::with_ft`, `temporal.cpp:77-95` + `combine` `:114-129` -> d [Q, N]."""
    s = np.asarray(seqs)
    mean = s.astype(np.complex128).mean(axis=-1, keepdims=True)
    t = s.astype(_CPLX[precision]) - mean.astype(_CPLX[precision])
    d_a = averages_term(t)
    corr = correlation(t, precision)
    n = s.shape[-1]
    ramp = (n - np.arange(n)).astype(np.float64)
    return d_a - 2.0 * corr / ramp


def direct_sequence(seqs: np.ndarray) -> np.ndarray:
    """`temporal.cpp:150-177` d only: O(N^2) defining loop, batch [Q, N], f64."""
    s = np.asarray(seqs, dtype=np.complex128)
    n = s.shape[-1]
    d = np.zeros(s.shape, dtype=np.float64)
    for m in range(n):
        diff = s[..., : n - m] - s[..., m:]
        d[..., m] = (diff.real ** 2 + diff.imag ** 2).sum(axis=-1) / (n - m)
    return d


# --------------------------------------------------------------------------- spatial


def spectra(stack: np.ndarray, precision: str = "f64") -> np.ndarray:
    """Per-frame half-plane spectra [N, H, W/2+1] (`SpatialTransform::run`)."""
    st = np.asarray(stack).astype(_REAL[precision])
    return np.fft.rfft2(st, axes=(-2, -1)).astype(_CPLX[precision], copy=False)


def normalize_lags(lags, frames: int):
    """`result_map.cpp:31-41` (+ `all_lags` :43-48 when empty)."""
    if lags is None or len(lags) == 0:
        return list(range(frames))
    out = sorted(int(x) for x in lags)
    for i, v in enumerate(out):
        if v < 0 or v >= frames:
            raise ValueError(f"lag {v} outside [0, {frames - 1}]")
        if i and out[i - 1] == v:
            raise ValueError(f"duplicate lag {v}")
    return out


def log_lags(frames: int):
    """`result_map.cpp:50-57`."""
    lags, m = [], 1
    while m < frames:
        lags.append(m)
        m <<= 1
    if frames > 1 and (not lags or lags[-1] != frames - 1):
        lags.append(frames - 1)
    return lags


def run_with_ft(stack: np.ndarray, precision: str = "f64", lags=None, q_max=None,
                chunk: int = 1 << 14) -> np.ndarray:
    """`ddm::run` WITH_FT (`scheduler.cpp:62-180`, `:413-483`) -> map [L, H, W/2+1] f64."""
    st = np.asarray(stack)
    n, h, w = st.shape
    lag_list = normalize_lags(lags, n)
    flat = cutoff_set(w, h, q_max)
    if flat.size == 0:
        raise ValueError("wave-vector cutoff retains nothing")
    sp = spectra(st, precision).reshape(n, -1)
    hc = half_cols(w)
    out = np.zeros((len(lag_list), h * hc), dtype=np.float64)
    li = np.asarray(lag_list)
    for b in range(0, flat.size, chunk):
        idx = flat[b:b + chunk]
        seq = np.ascontiguousarray(sp[:, idx].T)  # corner turn, `scheduler.cpp:122-126`
        d = with_ft(seq, precision)
        vals = d[:, li].T
        vals[li == 0] = 0.0                     # `scheduler.cpp:157-160`
        out[:, idx] = vals
    return out.reshape(len(lag_list), h, hc)


def run_without_ft(stack: np.ndarray, precision: str = "f64", lags=None, q_max=None):
    """WITHOUT_FT cross-check (`pairwise.cpp:11-72`): f64 accumulation of |S_{n-m}-S_n|^2."""
    st = np.asarray(stack)
    n, h, w = st.shape
    lag_list = normalize_lags(lags, n)
    flat = cutoff_set(w, h, q_max)
    sp = spectra(st, precision).reshape(n, -1)[:, flat].astype(np.complex128)
    hc = half_cols(w)
    out = np.zeros((len(lag_list), h * hc), dtype=np.float64)
    for i, m in enumerate(lag_list):
        if m == 0:
            continue
        diff = sp[: n - m] - sp[m:]
        out[i, flat] = (diff.real ** 2 + diff.imag ** 2).sum(axis=0) / (n - m)
    return out.reshape(len(lag_list), h, hc)


def azimuthal_average(values: np.ndarray, width: int, height: int, q_max=None):
    """`analysis.cpp:61-97`: ring means [L, bins] and counts [bins]."""
    v = np.asarray(values, dtype=np.float64).reshape(values.shape[0], -1)
    flat = cutoff_set(width, height, q_max)
    hc = half_cols(width)
    q = q_magnitude(flat // hc, flat % hc, height)
    # std::llround: halves away from zero (q >= 0)
    bins = np.floor(q + 0.5).astype(np.int64)
    nb = int(bins.max()) + 1
    counts = np.bincount(bins, minlength=nb).astype(np.int64)
    means = np.zeros((v.shape[0], nb))
    for li in range(v.shape[0]):
        means[li] = np.bincount(bins, weights=v[li, flat], minlength=nb)
    nz = counts > 0
    means[:, nz] /= counts[nz]
    return means, counts


def validate(values: np.ndarray, precision: str) -> None:
    """`ResultArchive::validate`, `archive.cpp:44-58`."""
    v = np.asarray(values)
    if not np.all(np.isfinite(v)):
        raise ValueError("result map contains non-finite values")
    peak = float(v.max()) if v.size else 0.0
    eps = 1e-4 if precision == "f32" else 1e-9
    if v.size and float(v.min()) < -eps * max(peak, 1.0):
        raise ValueError("result map contains negative values beyond tolerance")


def relative_deviation(a: np.ndarray, b: np.ndarray) -> float:
    """max|a-b| / global peak (`tests/unit/test_helpers.hpp:72-81`, `ddm_cli.cpp:132-141`)."""
    peak = max(float(np.abs(a).max(initial=0.0)), float(np.abs(b).max(initial=0.0)))
    diff = float(np.abs(np.asarray(a) - np.asarray(b)).max(initial=0.0))
    return diff / peak if peak > 0 else diff


def relative_l2(a: np.ndarray, b: np.ndarray) -> float:
    """||a-b||_2 / ||b||_2 — the north-star parity metric (BASELINE.json)."""
    nb = float(np.linalg.norm(np.asarray(b, dtype=np.float64).ravel()))
    d = float(np.linalg.norm((np.asarray(a, dtype=np.float64) - b).ravel()))
    return d / nb if nb > 0 else d


# --------------------------------------------------------------------------- inputs


def random_stack(width: int, height: int, frames: int, seed: int) -> np.ndarray:
    """Portable u16 random stack: mt19937_64 >> 48, frame-major [N, H, W]."""
    return (mt19937_64(seed, width * height * frames) >> np.uint64(48)).astype(
        np.uint16).reshape(frames, height, width)


def mt19937_64(seed: int, count: int) -> np.ndarray:
    """Reference-free MT19937-64 stream (the std::mt19937_64 definition), vectorised."""
    nn, mm = 312, 156
    a = np.uint64(0xB5026F5AA96619E9)
    upper, lower = np.uint64(0xFFFFFFFF80000000), np.uint64(0x7FFFFFFF)
    mt = np.zeros(nn, dtype=np.uint64)
    mt[0] = np.uint64(seed)
    with np.errstate(over="ignore"):
        for i in range(1, nn):
            prev = mt[i - 1]
            mt[i] = np.uint64(6364136223846793005) * (prev ^ (prev >> np.uint64(62))) + np.uint64(i)
    out = np.empty(count, dtype=np.uint64)
    filled = 0
    while filled < count:
        # twist, vectorised in the three dependency ranges of the in-place recurrence
        for lo, hi in ((0, nn - mm), (nn - mm, nn - 1), (nn - 1, nn)):
            i = np.arange(lo, hi)
            x = (mt[i] & upper) | (mt[(i + 1) % nn] & lower)
            xa = (x >> np.uint64(1)) ^ np.where(x & np.uint64(1), a, np.uint64(0))
            mt[i] = mt[(i + mm) % nn] ^ xa
        y = mt.copy()
        y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
        y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        y ^= y >> np.uint64(43)
        take = min(nn, count - filled)
        out[filled:filled + take] = y[:take]
        filled += take
    return out


def ramp_check() -> bool:
    """Hand-evaluated KAT (`test_temporal.cpp:90-98`): [1,2,3] -> d = [0, 1, 4]."""
    d = with_ft(np.array([[1, 2, 3]], dtype=np.complex128))[0]
    d[0] = 0.0
    return bool(np.allclose(d, [0, 1, 4], atol=1e-12))


def frames_per_second(frames: int, seconds: float) -> float:
    return frames / seconds if seconds > 0 else math.inf


# --------------------------------------------------------------------------- relaxation fits


def fit_exponential(t: np.ndarray, y: np.ndarray, frame_interval: float = 1.0):
    """`analysis.cpp:108-224`: Levenberg-Marquardt of y = A (1 - exp(-t / tau)) + B over
    (A, B, ln tau), sequential sums as the reference. Returns (A, B, tau, residual, flag) with
    flag 'ok' | 'degenerate' | 'no_converge'."""
    t = np.asarray(t, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if t.size < 4:
        raise ValueError("fit_exponential: need at least 4 usable lags")
    y_max, y_min = float(y.max()), float(y.min())
    scale = max(abs(y_max), abs(y_min), 1e-300)
    if y_max - y_min <= 1e-12 * scale:
        return 0.0, float(np.sum(y)) / y.size, frame_interval, 0.0, "degenerate"

    def cost(a, b, tau):
        s = 0.0
        for ti, yi in zip(t, y):
            r = a * (1.0 - np.exp(-ti / tau)) + b - yi
            s += r * r
        return s

    a, b = y_max, 0.0
    knee = a * (1.0 - np.exp(-1.0))
    tau = float(t[int(np.argmin(np.abs(y - knee)))])
    lam = 1e-3
    c = cost(a, b, tau)
    converged = False
    for _ in range(200):
        jtj = np.zeros((3, 3))
        jtr = np.zeros(3)
        for ti, yi in zip(t, y):
            e = np.exp(-ti / tau)
            r = a * (1.0 - e) + b - yi
            j = np.array([1.0 - e, 1.0, -a * e * ti / tau])
            jtj += np.outer(j, j)
            jtr += j * r
        damped = jtj.copy()
        for p in range(3):
            damped[p, p] += lam * max(jtj[p, p], 1e-300)
        try:
            if np.min(np.abs(np.linalg.eigvals(damped))) < 1e-300:
                raise np.linalg.LinAlgError
            step = np.linalg.solve(damped, -jtr)
        except np.linalg.LinAlgError:
            lam *= 5.0
            continue
        a2, b2 = a + step[0], b + step[1]
        tau2 = tau * np.exp(np.clip(step[2], -5.0, 5.0))
        c2 = cost(a2, b2, tau2)
        if c2 <= c:
            gain = c - c2
            a, b, tau, c = a2, b2, tau2, c2
            lam = max(lam / 3.0, 1e-12)
            if gain <= 1e-14 * (c + 1e-300):
                converged = True
                break
        else:
            lam *= 5.0
            if lam > 1e12:
                converged = True
                break
    return a, b, tau, float(np.sqrt(c / t.size)), "ok" if converged else "no_converge"


def estimate_diffusion(fits, width: int, q_lo: int, q_hi: int):
    """`analysis.cpp:242-271`: D from 1/tau = D q^2 (through the origin), q = 2 pi bin / width,
    over the 'ok' fits of bins [q_lo, q_hi]. fits: {bin: (A, B, tau, residual, flag)}."""
    sxx = sxy = 0.0
    used = 0
    for b, (_, _, tau, _, flag) in fits.items():
        if flag != "ok" or b < q_lo or b > q_hi:
            continue
        x = (2.0 * np.pi * b / width) ** 2
        sxx += x * x
        sxy += x / tau
        used += 1
    return (sxy / sxx if used and sxx > 0 else 0.0), used

"""ORACLE / TEST INFRASTRUCTURE ONLY — ctypes access to the unmodified reference library.

`oracle/_ref/libddmref.so` is the reference core (`/root/reference/proj/core/src/*.cpp`)
compiled by `oracle/Makefile` against our FFTW-API shim.  Only tests/, bench.py's
reference arm / cpu_baseline and __graft_entry__.smoke() may import this module, and only
as the checker or the timed CPU baseline — never on the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "_ref" / "libddmref.so"

_lib = None


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def available() -> bool:
    return LIB_PATH.exists()


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle`")
        _lib = C.CDLL(str(LIB_PATH))
        _lib.ref_pad_length.restype = C.c_int64
        _lib.ref_pad_length.argtypes = [C.c_int64]
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _check(rc, err):
    if rc != 0:
        raise RefError(rc, err.value.decode(errors="replace"))


def pad_length(n: int) -> int:
    v = lib().ref_pad_length(C.c_int64(n))
    if v < 0:
        raise RefError(1, "pad_length: sequence must have at least one frame")
    return int(v)


def _seq(seq):
    s = np.ascontiguousarray(np.asarray(seq, dtype=np.complex128))
    return s.view(np.float64), s.size


@dataclass
class LagProfile:
    d: np.ndarray
    d_a: np.ndarray
    corr: np.ndarray
    temporal_ffts: int = 0


def with_ft_sequence(seq, precision: str = "f64") -> LagProfile:
    inter, n = _seq(seq)
    d, da, c = (np.zeros(n) for _ in range(3))
    cnt = C.c_uint64(0)
    err = C.create_string_buffer(512)
    rc = lib().ref_with_ft_sequence(_p(inter, C.c_double), C.c_int64(n),
                                    0 if precision == "f32" else 1,
                                    _p(d, C.c_double), _p(da, C.c_double), _p(c, C.c_double),
                                    C.byref(cnt), err, 512)
    _check(rc, err)
    return LagProfile(d, da, c, int(cnt.value))


def correlation_term(seq, precision: str = "f64") -> np.ndarray:
    inter, n = _seq(seq)
    c = np.zeros(n)
    err = C.create_string_buffer(512)
    rc = lib().ref_correlation_term(_p(inter, C.c_double), C.c_int64(n),
                                    0 if precision == "f32" else 1, _p(c, C.c_double), err, 512)
    _check(rc, err)
    return c


def averages_term(seq, precision: str = "f64") -> np.ndarray:
    inter, n = _seq(seq)
    a = np.zeros(n)
    err = C.create_string_buffer(512)
    rc = lib().ref_averages_term(_p(inter, C.c_double), C.c_int64(n),
                                 0 if precision == "f32" else 1, _p(a, C.c_double), err, 512)
    _check(rc, err)
    return a


def direct_sequence_oracle(seq) -> LagProfile:
    inter, n = _seq(seq)
    d, da, c = (np.zeros(n) for _ in range(3))
    err = C.create_string_buffer(512)
    rc = lib().ref_direct_sequence_oracle(_p(inter, C.c_double), C.c_int64(n),
                                          _p(d, C.c_double), _p(da, C.c_double),
                                          _p(c, C.c_double), err, 512)
    _check(rc, err)
    return LagProfile(d, da, c)


def forward_spectrum(frame, width: int, height: int, precision: str = "f64") -> np.ndarray:
    f = np.ascontiguousarray(np.asarray(frame, dtype=np.float64).reshape(-1))
    out = np.zeros(height * (width // 2 + 1), dtype=np.complex128)
    err = C.create_string_buffer(512)
    rc = lib().ref_forward_spectrum(_p(f, C.c_double), width, height,
                                    0 if precision == "f32" else 1,
                                    _p(out.view(np.float64), C.c_double), err, 512)
    _check(rc, err)
    return out.reshape(height, width // 2 + 1)


def generate(width=64, height=64, frames=256, particles=100, diffusion=0.5, psf_sigma=1.0,
             amplitude=1000.0, background=100.0, frame_interval=1.0, seed=0) -> np.ndarray:
    out = np.zeros((frames, height, width), dtype=np.uint16)
    err = C.create_string_buffer(512)
    rc = lib().ref_generate(C.c_int64(particles), C.c_double(diffusion), C.c_double(psf_sigma),
                            C.c_double(amplitude), C.c_double(background), width, height,
                            frames, C.c_double(frame_interval), C.c_uint64(seed),
                            _p(out, C.c_uint16), err, 512)
    _check(rc, err)
    return out


def cutoff_set(width: int, height: int, q_max=None) -> np.ndarray:
    count = C.c_int64(0)
    err = C.create_string_buffer(512)
    has = 0 if q_max is None else 1
    qm = 0.0 if q_max is None else float(q_max)
    rc = lib().ref_cutoff_set(width, height, has, C.c_double(qm), C.byref(count), None, err, 512)
    _check(rc, err)
    flat = np.zeros(count.value, dtype=np.int64)
    rc = lib().ref_cutoff_set(width, height, has, C.c_double(qm), C.byref(count),
                              _p(flat, C.c_int64), err, 512)
    _check(rc, err)
    return flat


def plan_with_ft(q_count: int, frames: int, nbytes: int, precision: str = "f64"):
    cap, groups = C.c_int64(0), C.c_int64(0)
    err = C.create_string_buffer(512)
    rc = lib().ref_plan_with_ft(C.c_int64(q_count), C.c_int64(frames), C.c_int64(nbytes),
                                0 if precision == "f32" else 1, C.byref(cap), C.byref(groups),
                                err, 512)
    _check(rc, err)
    return int(cap.value), int(groups.value)


@dataclass
class RefArchive:
    values: np.ndarray            # lags x H x (W/2+1), f64
    lags: np.ndarray
    counters: dict
    timing: dict


def run(stack: np.ndarray, algorithm: str = "with_ft", precision: str = "f64", lags=(),
        q_max=None, memory_bytes: int = 1 << 40, workers: int = 2,
        frame_interval: float = 1.0) -> RefArchive:
    """ddm::run over a MemoryFrameSource (`proj/core/src/scheduler.cpp:413-483`)."""
    st = np.ascontiguousarray(stack, dtype=np.uint16)
    n, h, w = st.shape
    lag_arr = np.ascontiguousarray(np.asarray(lags, dtype=np.int64))
    n_out = len(lag_arr) if len(lag_arr) else n
    plane = h * (w // 2 + 1)
    values = np.zeros(n_out * plane)
    out_lags = np.zeros(max(n_out, 1), dtype=np.int64)
    n_lags = C.c_int64(0)
    counters = np.zeros(3, dtype=np.uint64)
    timing = np.zeros(6)
    err = C.create_string_buffer(1024)
    alg = {"with_ft": 0, "without_ft": 1, "direct": 2}[algorithm]
    rc = lib().ref_run(_p(st, C.c_uint16), w, h, n, C.c_double(frame_interval), alg,
                       0 if precision == "f32" else 1,
                       _p(lag_arr, C.c_int64) if len(lag_arr) else None,
                       C.c_int64(len(lag_arr)), 0 if q_max is None else 1,
                       C.c_double(0.0 if q_max is None else q_max), C.c_int64(memory_bytes),
                       workers, _p(values, C.c_double), C.c_int64(values.size),
                       _p(out_lags, C.c_int64), C.byref(n_lags),
                       _p(counters, C.c_uint64), _p(timing, C.c_double), err, 1024)
    _check(rc, err)
    k = n_lags.value
    return RefArchive(values[: k * plane].reshape(k, h, w // 2 + 1), out_lags[:k].copy(),
                      dict(zip(("spatial_ffts", "temporal_ffts", "pairs"),
                               map(int, counters))),
                      dict(zip(("disk", "step1", "step2", "merge", "other", "total"),
                               map(float, timing))))


def azimuthal_average(values: np.ndarray, lags, width: int, height: int, q_max=None):
    v = np.ascontiguousarray(values, dtype=np.float64)
    lag_arr = np.ascontiguousarray(np.asarray(lags, dtype=np.int64))
    cap = int(np.ceil(np.hypot(height / 2, width / 2))) + 2
    means = np.zeros(len(lag_arr) * cap)
    counts = np.zeros(cap, dtype=np.int64)
    nb = C.c_int64(0)
    err = C.create_string_buffer(512)
    rc = lib().ref_azimuthal(_p(v, C.c_double), _p(lag_arr, C.c_int64), C.c_int64(len(lag_arr)),
                             width, height, 0 if q_max is None else 1,
                             C.c_double(0.0 if q_max is None else q_max), _p(means, C.c_double),
                             _p(counts, C.c_int64), C.c_int64(cap), C.byref(nb), err, 512)
    _check(rc, err)
    b = nb.value
    return means[: len(lag_arr) * b].reshape(len(lag_arr), b), counts[:b].copy()


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def analyze(path: str, out_dir: str, fmt: str = "raw_stack", algorithm: str = "with_ft",
            precision: str = "f64", lags=(), q_max=None, memory_bytes: int = 1 << 40,
            workers: int = 2) -> None:
    """The `ddm analyze` artefacts (`proj/tools/ddm_cli.cpp:206-240` composition): d_m*.bin,
    index.json, radial.csv and fits.csv written by the reference library into out_dir."""
    lag_arr = np.ascontiguousarray(np.asarray(lags, dtype=np.int64))
    err = C.create_string_buffer(1024)
    rc = lib().ref_analyze(str(path).encode(), 1 if fmt == "pgm_dir" else 0,
                           {"with_ft": 0, "without_ft": 1, "direct": 2}[algorithm],
                           0 if precision == "f32" else 1,
                           _p(lag_arr, C.c_int64) if len(lag_arr) else None,
                           C.c_int64(len(lag_arr)), 0 if q_max is None else 1,
                           C.c_double(0.0 if q_max is None else q_max), C.c_int64(memory_bytes),
                           workers, str(out_dir).encode(), err, 1024)
    _check(rc, err)


def bench_sweep(frame_counts, sizes, algorithms=("with_ft", "without_ft"), workers=(2,),
                budgets=(), repetitions: int = 1, warmup: int = 0, out_csv: str = "bench.csv"):
    """The reference's `ddm bench` sweep (`proj/core/src/bench.cpp`): writes bench.csv,
    returns the crossover N* per size (None = never)."""
    ax = [np.ascontiguousarray(np.asarray(list(v), dtype=np.int32)) for v in
          (frame_counts, sizes, [{"with_ft": 0, "without_ft": 1, "direct": 2}[a] for a in algorithms],
           workers)]
    bud = np.ascontiguousarray(np.asarray(list(budgets), dtype=np.int64))
    xn = np.zeros(len(ax[1]), np.int32)
    err = C.create_string_buffer(1024)
    rc = lib().ref_bench_sweep(_p(ax[0], C.c_int), len(ax[0]), _p(ax[1], C.c_int), len(ax[1]),
                               _p(ax[2], C.c_int), len(ax[2]), _p(ax[3], C.c_int), len(ax[3]),
                               _p(bud, C.c_int64) if len(bud) else None, len(bud), repetitions,
                               warmup, str(out_csv).encode(), _p(xn, C.c_int), err, 1024)
    _check(rc, err)
    return {int(s): (int(n) if n >= 0 else None) for s, n in zip(ax[1], xn)}

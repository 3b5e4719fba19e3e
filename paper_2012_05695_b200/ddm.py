"""Python view of the ddm-b200 C-ABI (include/ddm_b200.h), mirroring the reference API.

Names and argument meaning follow the reference C++ library (`proj/core/include/ddm/*.hpp`):
`run(stack, RunConfig)` is `ddm::run` over a MemoryFrameSource, `with_ft_sequence` is the
per-sequence engine, errors are `InputError` / `PlanError` / `IoError` (plus `DeviceError`).
All compute happens in `libddm_b200.so` on the GPU; there is no CPU fallback — if the
library is missing this module raises on first use.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, field
from pathlib import Path
from typing import Callable, Optional, Sequence

import numpy as np

# DDM_B200_LIB: another build of the library (A/B timing of kernel variants); default in-tree
LIB_PATH = Path(os.environ.get("DDM_B200_LIB") or Path(__file__).resolve().parent / "libddm_b200.so")


class Error(RuntimeError):
    """ddm::Error"""


class InputError(Error):
    """ddm::InputError (status 1)"""


class PlanError(Error):
    """ddm::PlanError (status 2)"""


class IoError(Error):
    """ddm::IoError (status 3)"""


class DeviceError(Error):
    """device failure (status 4)"""


_ERR = {1: InputError, 2: PlanError, 3: IoError, 4: DeviceError, 5: Error}


class Counters(C.Structure):
    _fields_ = [("spatial_ffts", C.c_uint64), ("temporal_ffts", C.c_uint64), ("pairs", C.c_uint64)]


class Timing(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("disk", "step1", "step2", "merge", "other", "total")]


BEFORE_MERGE = C.CFUNCTYPE(None, C.c_char_p, C.c_void_p)


class _RunConfig(C.Structure):
    _fields_ = [("algorithm", C.c_int), ("precision", C.c_int), ("lags", C.POINTER(C.c_int64)),
                ("n_lags", C.c_int64), ("has_q_max", C.c_int), ("q_max", C.c_double),
                ("memory_bytes", C.c_int64), ("workers", C.c_int), ("out_dir", C.c_char_p),
                ("before_merge", BEFORE_MERGE), ("before_merge_user", C.c_void_p),
                ("device", C.c_int)]


_lib = None


def lib():
    """Load the native library (raises if it was not built — no silent fallback)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2012_05695_b200.build`")
        L = C.CDLL(str(LIB_PATH))
        L.ddm_b200_last_error.restype = C.c_char_p
        L.ddm_b200_pad_length.restype = C.c_int64
        L.ddm_b200_pad_length.argtypes = [C.c_int64]
        L.ddm_b200_max_frames.restype = C.c_int64
        L.ddm_b200_max_frames.argtypes = [C.c_int]
        L.ddm_b200_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.ddm_b200_destroy.argtypes = [C.c_void_p]
        L.ddm_b200_stage_frames.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int]
        L.ddm_b200_stage_frames_u8.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int]
        L.ddm_b200_run_with_ft.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                           C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
        L.ddm_b200_session_engines.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
        L.ddm_b200_run_device.argtypes = [
            C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int64),
            C.c_int64, C.c_int, C.c_double, C.c_void_p, C.c_int, C.c_int, C.c_void_p,
            C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int)]
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib().ddm_b200_last_error().decode(errors="replace")
        raise _ERR.get(rc, Error)(msg)


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def device_count() -> int:
    n = C.c_int(0)
    _check(lib().ddm_b200_device_count(C.byref(n)))
    return n.value


def last_engines(device: int = 0) -> str:
    """The kernels the last run on `device` selected ("spatial=... temporal=...")."""
    buf = C.create_string_buffer(256)
    _check(lib().ddm_b200_last_engines(device, buf, C.c_int64(256)))
    return buf.value.decode()


def pad_length(n: int) -> int:
    v = lib().ddm_b200_pad_length(n)
    if v < 0:
        raise InputError("pad_length: sequence must have at least one frame")
    return int(v)


def max_frames(precision: str = "f32") -> int:
    return int(lib().ddm_b200_max_frames(0 if precision == "f32" else 1))


def half_cols(width: int) -> int:
    return width // 2 + 1


def plan_with_ft(q_count: int, frames: int, nbytes: int, precision: str = "f64"):
    cap, groups = C.c_int64(0), C.c_int64(0)
    _check(lib().ddm_b200_plan_with_ft(C.c_int64(q_count), C.c_int64(frames), C.c_int64(nbytes),
                                       0 if precision == "f32" else 1, C.byref(cap), C.byref(groups)))
    return int(cap.value), int(groups.value)


def cutoff_set(width: int, height: int, q_max: Optional[float] = None) -> np.ndarray:
    count = C.c_int64(0)
    has, qm = (0, 0.0) if q_max is None else (1, float(q_max))
    _check(lib().ddm_b200_cutoff_set(width, height, has, C.c_double(qm), C.byref(count), None))
    flat = np.zeros(count.value, dtype=np.int64)
    _check(lib().ddm_b200_cutoff_set(width, height, has, C.c_double(qm), C.byref(count),
                                     _p(flat, C.c_int64)))
    return flat


@dataclass
class RunConfig:
    """ddm::RunConfig (`scheduler.hpp:78-93`)."""
    algorithm: str = "with_ft"
    precision: str = "f64"
    lags: Sequence[int] = ()
    q_max: Optional[float] = None
    memory_bytes: int = 0
    workers: int = 2
    out_dir: Optional[str] = None
    before_merge: Optional[Callable[[str], None]] = None
    device: int = 0


@dataclass
class ResultArchive:
    """ddm::ResultArchive: map values lag-major [lags, H, W/2+1] f64."""
    values: np.ndarray
    lags: np.ndarray
    width: int
    height: int
    frames: int
    frame_interval: float
    algorithm: str
    precision: str
    q_max: Optional[float]
    workers: int
    counters: dict = field(default_factory=dict)
    timing: dict = field(default_factory=dict)

    def lag_plane(self, i: int) -> np.ndarray:
        return self.values[i]

    def lag_index(self, lag: int) -> int:
        idx = np.searchsorted(self.lags, lag)
        return int(idx) if idx < len(self.lags) and self.lags[idx] == lag else -1


def _config(cfg: RunConfig, keep):
    alg = {"with_ft": 0, "without_ft": 1, "direct": 2}.get(cfg.algorithm)
    if alg is None:
        raise InputError(f"unknown algorithm '{cfg.algorithm}'")
    if cfg.precision not in ("f32", "f64"):
        raise InputError(f"unknown precision '{cfg.precision}'")
    lags = np.ascontiguousarray(np.asarray(list(cfg.lags), dtype=np.int64))
    keep.append(lags)
    c = _RunConfig()
    c.algorithm = alg
    c.precision = 0 if cfg.precision == "f32" else 1
    c.lags = _p(lags, C.c_int64) if len(lags) else None
    c.n_lags = len(lags)
    c.has_q_max = 0 if cfg.q_max is None else 1
    c.q_max = 0.0 if cfg.q_max is None else float(cfg.q_max)
    c.memory_bytes = int(cfg.memory_bytes)
    c.workers = int(cfg.workers)
    c.out_dir = cfg.out_dir.encode() if cfg.out_dir else None
    if cfg.before_merge is not None:
        user_fn = cfg.before_merge
        errors = []

        def tramp(ws, _user):
            try:
                user_fn(ws.decode())
            except Exception as e:  # pragma: no cover - surfaced below
                errors.append(e)
        cb = BEFORE_MERGE(tramp)
        keep.append(cb)
        keep.append(errors)
        c.before_merge = cb
    else:
        c.before_merge = BEFORE_MERGE()
    c.before_merge_user = None
    c.device = int(cfg.device)
    return c


def run(stack, config: RunConfig, frame_interval: float = 1.0) -> ResultArchive:
    """ddm::run (`scheduler.cpp:413-483`) on a frame-major [N, H, W] uint16 (or uint8) stack."""
    st = np.asarray(stack)
    if st.ndim != 3:
        raise InputError("stack must be [frames, height, width]")
    u8 = st.dtype == np.uint8
    st = np.ascontiguousarray(st, dtype=np.uint8 if u8 else np.uint16)
    n, h, w = st.shape
    n_out = len(config.lags) if len(config.lags) else n
    plane = h * half_cols(w)
    values = np.empty(max(n_out, 1) * plane)
    out_lags = np.zeros(max(n_out, 1), dtype=np.int64)
    n_lags = C.c_int64(0)
    counters, timing = Counters(), Timing()
    keep: list = []
    c = _config(config, keep)
    fn = lib().ddm_b200_run_u8 if u8 else lib().ddm_b200_run_u16
    rc = fn(_p(st, C.c_uint8 if u8 else C.c_uint16), w, h, n, C.c_double(frame_interval),
            C.byref(c), _p(values, C.c_double), C.c_int64(values.size), _p(out_lags, C.c_int64),
            C.byref(n_lags), C.byref(counters), C.byref(timing))
    for item in keep:
        if isinstance(item, list) and item and isinstance(item[0], Exception):
            raise item[0]
    _check(rc)
    k = n_lags.value
    return ResultArchive(values[: k * plane].reshape(k, h, half_cols(w)), out_lags[:k].copy(), w, h,
                         n, frame_interval, config.algorithm,
                         "f64" if config.algorithm == "direct" else config.precision, config.q_max,
                         config.workers,
                         {f: int(getattr(counters, f)) for f, _ in Counters._fields_},
                         {f: float(getattr(timing, f)) for f, _ in Timing._fields_})


class Session:
    """Opaque staging session (`ddm_b200_create` / `_stage_frames` / `_run_with_ft`,
    SURVEY.md §8b): one stack resident in HBM, any number of WITH_FT runs over it, each with
    the reference WithFt branch's contract (`scheduler.cpp:413-483`). Owns its own device
    engine, so sessions on one GPU run concurrently; use one from one thread at a time."""

    def __init__(self, width: int, height: int, frames: int, precision: str = "f32", device: int = 0):
        if precision not in ("f32", "f64"):
            raise InputError(f"unknown precision '{precision}'")
        self.width, self.height, self.frames = int(width), int(height), int(frames)
        h = C.c_void_p()
        _check(lib().ddm_b200_create(self.width, self.height, self.frames,
                                     0 if precision == "f32" else 1, int(device), C.byref(h)))
        self._h = h

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            _check(lib().ddm_b200_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def stage(self, frames, first: int = 0) -> None:
        """frames [first, first + len(frames)) from a [count, H, W] uint16 or uint8 array"""
        st = np.asarray(frames)
        if st.ndim != 3 or st.shape[1:] != (self.height, self.width):
            raise InputError("frames must be [count, height, width] of the session's frame size")
        u8 = st.dtype == np.uint8
        st = np.ascontiguousarray(st, dtype=np.uint8 if u8 else np.uint16)
        fn = lib().ddm_b200_stage_frames_u8 if u8 else lib().ddm_b200_stage_frames
        _check(fn(self._h, _p(st, C.c_uint8 if u8 else C.c_uint16), int(first), int(st.shape[0])))

    def run_with_ft(self, wave_vectors=None, lags=()):
        """-> (map [n_lags, H, W/2+1] f64, counters, timing). wave_vectors: ascending flat
        indices (None = the whole half plane); lags: empty = every lag."""
        plane = self.height * half_cols(self.width)
        wv = None if wave_vectors is None else np.ascontiguousarray(np.asarray(wave_vectors), dtype=np.int64)
        lg = np.ascontiguousarray(np.asarray(list(lags), dtype=np.int64))
        n_out = len(np.unique(lg)) if len(lg) else self.frames
        values = np.empty(max(n_out, 1) * plane)
        counters, timing = Counters(), Timing()
        _check(lib().ddm_b200_run_with_ft(
            self._h, _p(wv, C.c_int64) if wv is not None else None,
            C.c_int64(0 if wv is None else wv.size), _p(lg, C.c_int64) if len(lg) else None,
            C.c_int64(len(lg)), _p(values, C.c_double), C.c_int64(values.size), C.byref(counters),
            C.byref(timing)))
        return (values[: n_out * plane].reshape(n_out, self.height, half_cols(self.width)),
                {f: int(getattr(counters, f)) for f, _ in Counters._fields_},
                {f: float(getattr(timing, f)) for f, _ in Timing._fields_})

    def engines(self) -> str:
        buf = C.create_string_buffer(256)
        _check(lib().ddm_b200_session_engines(self._h, buf, C.c_int64(256)))
        return buf.value.decode()


def run_raw_stack(path: str, config: RunConfig) -> ResultArchive:
    """ddm::run over a RawStackFileSource (`frame_source.cpp:27-78`)."""
    with open(path, "rb") as f:
        import json
        hdr = json.loads(f.readline())
    n, h, w = int(hdr["frames"]), int(hdr["height"]), int(hdr["width"])
    n_out = len(config.lags) if len(config.lags) else n
    plane = h * half_cols(w)
    values = np.empty(max(n_out, 1) * plane)
    out_lags = np.zeros(max(n_out, 1), dtype=np.int64)
    n_lags = C.c_int64(0)
    counters, timing = Counters(), Timing()
    keep: list = []
    c = _config(config, keep)
    rc = lib().ddm_b200_run_raw_stack(str(path).encode(), C.byref(c), _p(values, C.c_double),
                                      C.c_int64(values.size), _p(out_lags, C.c_int64),
                                      C.byref(n_lags), C.byref(counters), C.byref(timing))
    _check(rc)
    k = n_lags.value
    return ResultArchive(values[: k * plane].reshape(k, h, half_cols(w)), out_lags[:k].copy(), w, h,
                         n, float(hdr.get("frame_interval", 1.0)), config.algorithm,
                         config.precision, config.q_max, config.workers,
                         {f: int(getattr(counters, f)) for f, _ in Counters._fields_},
                         {f: float(getattr(timing, f)) for f, _ in Timing._fields_})


def load_stack(path: str, fmt: str = "raw_stack") -> np.ndarray:
    """ddm::load_stack (raw_stack | pgm_dir) -> [N, H, W] uint16 (host only)."""
    f = {"raw_stack": 0, "pgm_dir": 1}.get(fmt)
    if f is None:
        raise InputError(f"unknown stack format '{fmt}'")
    w, h, n = C.c_int(0), C.c_int(0), C.c_int(0)
    _check(lib().ddm_b200_stack_dims(str(path).encode(), f, C.byref(w), C.byref(h), C.byref(n)))
    out = np.empty((n.value, h.value, w.value), dtype=np.uint16)
    _check(lib().ddm_b200_load_stack(str(path).encode(), f, _p(out, C.c_uint16), C.c_int64(out.size)))
    return out


def run_pgm_dir(path: str, config: RunConfig) -> ResultArchive:
    """ddm::run over a PgmDirSource (`frame_source.cpp:80-95`)."""
    w, h, n = C.c_int(0), C.c_int(0), C.c_int(0)
    _check(lib().ddm_b200_stack_dims(str(path).encode(), 1, C.byref(w), C.byref(h), C.byref(n)))
    w, h, n = w.value, h.value, n.value
    n_out = len(config.lags) if len(config.lags) else n
    plane = h * half_cols(w)
    values = np.empty(max(n_out, 1) * plane)
    out_lags = np.zeros(max(n_out, 1), dtype=np.int64)
    n_lags = C.c_int64(0)
    counters, timing = Counters(), Timing()
    keep: list = []
    c = _config(config, keep)
    _check(lib().ddm_b200_run_pgm_dir(str(path).encode(), C.byref(c), _p(values, C.c_double),
                                      C.c_int64(values.size), _p(out_lags, C.c_int64),
                                      C.byref(n_lags), C.byref(counters), C.byref(timing)))
    k = n_lags.value
    return ResultArchive(values[: k * plane].reshape(k, h, half_cols(w)), out_lags[:k].copy(), w, h,
                         n, 1.0, config.algorithm,
                         "f64" if config.algorithm == "direct" else config.precision, config.q_max,
                         config.workers,
                         {f: int(getattr(counters, f)) for f, _ in Counters._fields_},
                         {f: float(getattr(timing, f)) for f, _ in Timing._fields_})


def analyze(path: str, out: str, config: RunConfig, fmt: str = "auto", lag_spec: str = "all",
            memory_limit: Optional[str] = None) -> dict:
    """`ddm analyze` (`tools/ddm_cli.cpp:206-240`): run, write_results, radial.csv, fits.csv
    (one C-ABI call, ddm_b200_analyze) and the CLI's run.json option echo (`:189-203`).

    `config.lags` is the resolved lag list; `lag_spec` / `memory_limit` are only echoed."""
    f = {"raw_stack": 0, "pgm_dir": 1, "auto": -1}.get(fmt)
    if f is None:
        raise InputError(f"unknown stack format '{fmt}'")
    os.makedirs(out, exist_ok=True)
    keep: list = []
    c = _config(config, keep)
    n_lags, fits = C.c_int64(0), C.c_int64(0)
    counters, timing = Counters(), Timing()
    rc = lib().ddm_b200_analyze(str(path).encode(), f, C.byref(c), str(out).encode(), C.byref(n_lags),
                                C.byref(fits), C.byref(counters), C.byref(timing))
    for item in keep:
        if isinstance(item, list) and item and isinstance(item[0], Exception):
            raise item[0]
    _check(rc)
    resolved = fmt if fmt != "auto" else ("pgm_dir" if os.path.isdir(path) else "raw_stack")
    echo = {"tool_version": "0.1.0-b200", "input": str(path), "format": resolved, "lags": lag_spec,
            "q_max": config.q_max, "memory_limit_bytes": int(config.memory_bytes),
            "workers": int(config.workers), "precision": config.precision, "out": str(out),
            "subcommand": "analyze", "algorithm": config.algorithm}
    with open(os.path.join(out, "run.json"), "w") as fh:
        json.dump(echo, fh, indent=2, sort_keys=True)
        fh.write("\n")
    return {"n_lags": n_lags.value, "fits_written": bool(fits.value),
            "counters": {k: int(getattr(counters, k)) for k, _ in Counters._fields_},
            "timing": {k: float(getattr(timing, k)) for k, _ in Timing._fields_}}


def bench_sweep(frame_counts, sizes, algorithms=("with_ft", "without_ft"), workers=(2,),
                budgets=(), repetitions: int = 3, warmup: int = 1, out: Optional[str] = None):
    """`ddm bench` (`tools/ddm_cli.cpp:338-385`, `core/src/bench.cpp`): the sweep over
    synthetic stacks through one C-ABI call (ddm_b200_bench_sweep), bench.csv in `out`, plus
    the CLI's run.json echo. Returns (rows of bench.csv as dicts, {size: N* or None})."""
    import csv
    import tempfile
    alg_ids = []
    for a in algorithms:
        if a not in ("with_ft", "without_ft", "direct"):
            raise InputError(f"unknown algorithm '{a}'")
        alg_ids.append({"with_ft": 0, "without_ft": 1, "direct": 2}[a])
    ax = [np.ascontiguousarray(np.asarray(list(v), dtype=np.int32)) for v in (frame_counts, sizes, alg_ids, workers)]
    bud = np.ascontiguousarray(np.asarray(list(budgets), dtype=np.int64))
    ns = max(len(ax[1]), 1)
    xs, xn, nx = np.zeros(ns, np.int32), np.zeros(ns, np.int32), C.c_int(0)
    tmp = None
    if out is None:
        tmp = tempfile.TemporaryDirectory()
        out = tmp.name
    os.makedirs(out, exist_ok=True)
    csv_path = os.path.join(out, "bench.csv")

    def ptr(a, ct):
        return _p(a, ct) if len(a) else None
    _check(lib().ddm_b200_bench_sweep(ptr(ax[0], C.c_int), len(ax[0]), ptr(ax[1], C.c_int), len(ax[1]),
                                      ptr(ax[2], C.c_int), len(ax[2]), ptr(ax[3], C.c_int), len(ax[3]),
                                      ptr(bud, C.c_int64), len(bud), int(repetitions), int(warmup),
                                      csv_path.encode(), _p(xs, C.c_int), _p(xn, C.c_int), C.byref(nx)))
    with open(csv_path, newline="") as f:
        rows = list(csv.DictReader(f))
    echo = {"subcommand": "bench", "tool_version": "0.1.0-b200",
            "sweep": ",".join(str(n) for n in frame_counts), "sizes": ",".join(str(s) for s in sizes),
            "algorithms": ",".join(algorithms), "workers": ",".join(str(w) for w in workers),
            "budgets": ",".join(str(b) for b in budgets) if len(budgets) else "default",
            "repetitions": int(repetitions), "warmup": int(warmup), "out": str(out)}
    with open(os.path.join(out, "run.json"), "w") as fh:
        json.dump(echo, fh, indent=2, sort_keys=True)
        fh.write("\n")
    if tmp is not None:
        tmp.cleanup()
    return rows, {int(xs[i]): (int(xn[i]) if xn[i] >= 0 else None) for i in range(nx.value)}


def compare(path: str, config: RunConfig, algorithms=("with_ft", "without_ft"), fmt: str = "auto",
            out: Optional[str] = None) -> dict:
    """`ddm compare` (`tools/ddm_cli.cpp:247-290`) through ddm_b200_compare; with `out`, the
    CLI's compare.json report is written there."""
    ids = {"with_ft": 0, "without_ft": 1, "direct": 2}
    if len(algorithms) != 2:
        raise InputError("--algorithms needs exactly two names")
    for a in algorithms:
        if a not in ids:
            raise InputError(f"unknown algorithm '{a}'")
    f = {"raw_stack": 0, "pgm_dir": 1, "auto": -1}.get(fmt)
    if f is None:
        raise InputError(f"unknown stack format '{fmt}'")
    keep: list = []
    c = _config(config, keep)
    dev, tol, ok = C.c_double(0.0), C.c_double(0.0), C.c_int(0)
    ta, tb = Timing(), Timing()
    _check(lib().ddm_b200_compare(str(path).encode(), f, C.byref(c), ids[algorithms[0]], ids[algorithms[1]],
                                  C.byref(dev), C.byref(tol), C.byref(ok), C.byref(ta), C.byref(tb)))
    resolved = fmt if fmt != "auto" else ("pgm_dir" if os.path.isdir(path) else "raw_stack")
    report = {"subcommand": "compare", "tool_version": "0.1.0-b200", "input": str(path),
              "format": resolved, "algorithms": list(algorithms), "precision": config.precision,
              "deviation": dev.value, "tolerance": tol.value, "pass": bool(ok.value)}
    if out:
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, "compare.json"), "w") as fh:
            json.dump(report, fh, indent=2, sort_keys=True)
            fh.write("\n")
    report["timing"] = [{k: float(getattr(t, k)) for k, _ in Timing._fields_} for t in (ta, tb)]
    return report


def crossover(cells) -> dict:
    """ddm::crossover (`core/src/bench.cpp:144-183`) on [(algorithm, N, size, seconds_total,
    failed), ...]: {size: N* or None}."""
    ids = {"with_ft": 0, "without_ft": 1, "direct": 2}
    n = len(cells)
    alg = np.asarray([ids[c[0]] for c in cells], np.int32)
    fr = np.asarray([c[1] for c in cells], np.int32)
    sz = np.asarray([c[2] for c in cells], np.int32)
    tot = np.asarray([c[3] for c in cells], np.float64)
    fail = np.asarray([1 if (len(c) > 4 and c[4]) else 0 for c in cells], np.int32)
    out_s, out_n, cnt = np.zeros(max(n, 1), np.int32), np.zeros(max(n, 1), np.int32), C.c_int(0)
    _check(lib().ddm_b200_crossover(C.c_int64(n), _p(alg, C.c_int), _p(fr, C.c_int), _p(sz, C.c_int),
                                    _p(tot, C.c_double), _p(fail, C.c_int), _p(out_s, C.c_int),
                                    _p(out_n, C.c_int), C.byref(cnt)))
    return {int(out_s[i]): (int(out_n[i]) if out_n[i] >= 0 else None) for i in range(cnt.value)}


def synth(out: str, size: int = 64, frames: int = 256, particles: int = 100, diffusion: float = 0.5,
          psf_sigma: float = 1.0, amplitude: float = 1000.0, background: float = 100.0,
          frame_interval: float = 1.0, seed: int = 0) -> str:
    """`ddm synth` (`tools/ddm_cli.cpp:306-327`): out/stack.raw + out/synth.json. Returns the
    stack path."""
    _check(lib().ddm_b200_synth(str(out).encode(), C.c_int64(particles), C.c_double(diffusion),
                                C.c_double(psf_sigma), C.c_double(amplitude), C.c_double(background),
                                int(size), int(frames), C.c_double(frame_interval), C.c_uint64(seed)))
    return os.path.join(out, "stack.raw")


@dataclass
class LagProfile:
    d: np.ndarray
    d_a: np.ndarray
    corr: np.ndarray


def sequences_with_ft(seqs, precision: str = "f64", device: int = 0, terms: bool = False):
    """Batched SequenceEngine<S>::with_ft on the GPU: seqs [Q, N] complex -> d [Q, N] (and
    d_a, corr restored to the original basis when terms=True)."""
    s = np.ascontiguousarray(np.atleast_2d(np.asarray(seqs, dtype=np.complex128)))
    q, n = s.shape
    d = np.empty((q, n))
    d_a = np.empty((q, n)) if terms else None
    corr = np.empty((q, n)) if terms else None
    cnt = C.c_uint64(0)
    _check(lib().ddm_b200_sequences_with_ft(
        _p(s.view(np.float64), C.c_double), C.c_int64(q), C.c_int64(n),
        0 if precision == "f32" else 1, device, _p(d, C.c_double),
        _p(d_a, C.c_double) if terms else None, _p(corr, C.c_double) if terms else None,
        C.byref(cnt)))
    return (d, d_a, corr) if terms else d


def with_ft_sequence(seq, precision: str = "f64") -> LagProfile:
    """ddm::with_ft_sequence<S> (`temporal.cpp:141-148`)."""
    d, d_a, corr = sequences_with_ft(np.asarray(seq)[None, :], precision, terms=True)
    return LagProfile(d[0], d_a[0], corr[0])


def compute_spectra(stack, precision: str = "f64", device: int = 0) -> np.ndarray:
    """ddm::compute_spectra (`spectrum.cpp:29-63`): [N, H, W/2+1] complex128."""
    st = np.ascontiguousarray(stack, dtype=np.uint16)
    n, h, w = st.shape
    out = np.empty((n, h, half_cols(w)), dtype=np.complex128)
    _check(lib().ddm_b200_spectra_u16(_p(st, C.c_uint16), w, h, n, 0 if precision == "f32" else 1,
                                      device, _p(out.view(np.float64), C.c_double)))
    return out


def forward_spectrum(frame, width: int, height: int, precision: str = "f64") -> np.ndarray:
    """ddm::forward_spectrum (`spectrum.cpp:12-27`): [H, W/2+1] complex128."""
    f = np.ascontiguousarray(np.asarray(frame, dtype=np.float64).reshape(-1))
    out = np.empty((height, half_cols(width)), dtype=np.complex128)
    _check(lib().ddm_b200_forward_spectrum(_p(f, C.c_double), width, height,
                                           0 if precision == "f32" else 1, 0,
                                           _p(out.view(np.float64), C.c_double)))
    return out


def azimuthal_average(values, width: int, height: int, q_max: Optional[float] = None, device: int = 0):
    """ddm::azimuthal_average (`analysis.cpp:61-97`) -> (means [L, bins], counts [bins])."""
    v = np.ascontiguousarray(values, dtype=np.float64)
    L = v.shape[0]
    cap = int(np.ceil(np.hypot(height / 2, width / 2))) + 2
    means = np.zeros(L * cap)
    counts = np.zeros(cap, dtype=np.int64)
    nb = C.c_int64(0)
    _check(lib().ddm_b200_azimuthal(_p(v, C.c_double), C.c_int64(L), width, height,
                                    0 if q_max is None else 1,
                                    C.c_double(0.0 if q_max is None else q_max), device,
                                    _p(means, C.c_double), _p(counts, C.c_int64), C.c_int64(cap),
                                    C.byref(nb)))
    b = nb.value
    return means[: L * b].reshape(L, b), counts[:b].copy()


def run_azimuthal(stack, config: RunConfig):
    """ddm::run + ddm::azimuthal_average in one device pass (what `ddm analyze` computes,
    `ddm_cli.cpp:218-225`), ring sums fused into the temporal kernel where the register engines
    apply. Returns (means [L, bins], counts [bins], lags)."""
    st = np.ascontiguousarray(np.asarray(stack), dtype=np.uint16)
    if st.ndim != 3:
        raise InputError("stack must be [frames, height, width]")
    n, h, w = st.shape
    keep: list = []
    c = _config(config, keep)
    nb = C.c_int64(0)
    n_out = len(config.lags) if len(config.lags) else n
    out_lags = np.zeros(max(n_out, 1), dtype=np.int64)
    nl = C.c_int64(0)
    _check(lib().ddm_b200_run_azimuthal_u16(_p(st, C.c_uint16), w, h, n, C.byref(c), None,
                                            C.c_int64(0), None, C.byref(nb), _p(out_lags, C.c_int64),
                                            C.byref(nl)))
    b = nb.value
    means = np.zeros(max(nl.value, 1) * b)
    counts = np.zeros(b, dtype=np.int64)
    _check(lib().ddm_b200_run_azimuthal_u16(_p(st, C.c_uint16), w, h, n, C.byref(c),
                                            _p(means, C.c_double), C.c_int64(b),
                                            _p(counts, C.c_int64), C.byref(nb),
                                            _p(out_lags, C.c_int64), C.byref(nl)))
    k = nl.value
    return means[: k * b].reshape(k, b), counts, out_lags[:k].copy()


def run_azimuthal_device(frames_ptr: int, pixel_bytes: int, width: int, height: int, frames: int,
                         means_ptr: int, capacity: int, precision: str = "f32", lags=None,
                         q_max: Optional[float] = None, device: int = 0, stream: int = 0):
    """Device-resident run + ring average: means [L][capacity] f64 at means_ptr (HBM).
    Returns (bin_count, spatial_ms, temporal_ms, fused)."""
    lag_arr = np.ascontiguousarray(np.asarray(lags if lags is not None else [], dtype=np.int64))
    nb, sp, tp, fu = C.c_int64(0), C.c_double(0), C.c_double(0), C.c_int(0)
    _check(lib().ddm_b200_run_azimuthal_device(
        C.c_void_p(frames_ptr), pixel_bytes, width, height, frames,
        0 if precision == "f32" else 1, _p(lag_arr, C.c_int64) if len(lag_arr) else None,
        C.c_int64(len(lag_arr)), 0 if q_max is None else 1,
        C.c_double(0.0 if q_max is None else q_max), C.c_void_p(means_ptr), C.c_int64(capacity),
        None, C.byref(nb), device, C.c_void_p(stream), C.byref(sp), C.byref(tp), C.byref(fu)))
    return nb.value, sp.value, tp.value, bool(fu.value)


FIT_FLAGS = {0: "ok", 1: "degenerate", 2: "no_converge", -1: "not_fitted"}


def fit_rings(means, lags, counts, frame_interval: float = 1.0, device: int = 0):
    """ddm::fit_all_bins (`analysis.cpp:108-224`) on the device: per-ring
    (amplitude, baseline, tau, residual, flag) arrays over the profile's bins."""
    m = np.ascontiguousarray(means, dtype=np.float64)
    lg = np.ascontiguousarray(lags, dtype=np.int64)
    ct = np.ascontiguousarray(counts, dtype=np.int64)
    nb = m.shape[1]
    out = [np.zeros(nb) for _ in range(4)]
    flag = np.zeros(nb, dtype=np.int32)
    _check(lib().ddm_b200_fit_rings(_p(m, C.c_double), _p(lg, C.c_int64), C.c_int64(len(lg)),
                                    _p(ct, C.c_int64), C.c_int64(nb), C.c_double(frame_interval),
                                    device, *[_p(o, C.c_double) for o in out], _p(flag, C.c_int)))
    return out[0], out[1], out[2], out[3], flag


def estimate_diffusion(tau, flag, width: int, q_lo: int, q_hi: int):
    """ddm::estimate_diffusion (`analysis.cpp:242-271`) -> (coefficient, bins_used)."""
    t = np.ascontiguousarray(tau, dtype=np.float64)
    f = np.ascontiguousarray(flag, dtype=np.int32)
    coef, used = C.c_double(0.0), C.c_int64(0)
    _check(lib().ddm_b200_estimate_diffusion(_p(t, C.c_double), _p(f, C.c_int), C.c_int64(len(t)),
                                             C.c_int64(width), C.c_int64(q_lo), C.c_int64(q_hi),
                                             C.byref(coef), C.byref(used)))
    return coef.value, used.value


def generate(width=64, height=64, frames=256, particles=100, diffusion=0.5, psf_sigma=1.0,
             amplitude=1000.0, background=100.0, frame_interval=1.0, seed=0) -> np.ndarray:
    """ddm::generate (`synth.cpp:98-132`), bit-identical frames [N, H, W] uint16."""
    out = np.empty((frames, height, width), dtype=np.uint16)
    _check(lib().ddm_b200_generate(C.c_int64(particles), C.c_double(diffusion),
                                   C.c_double(psf_sigma), C.c_double(amplitude),
                                   C.c_double(background), width, height, frames,
                                   C.c_double(frame_interval), C.c_uint64(seed),
                                   _p(out, C.c_uint16)))
    return out


def generate_device(out_ptr: int, width=64, height=64, frames=256, particles=100, diffusion=0.5,
                    psf_sigma=1.0, amplitude=1000.0, background=100.0, frame_interval=1.0, seed=0,
                    device: int = 0, stream: int = 0) -> None:
    """ddm::generate rendered on the device into out_ptr ([frames][height][width] u16 in HBM,
    e.g. a torch tensor's data_ptr); the trajectories are the reference's draw sequence."""
    _check(lib().ddm_b200_generate_device(C.c_int64(particles), C.c_double(diffusion),
                                          C.c_double(psf_sigma), C.c_double(amplitude),
                                          C.c_double(background), width, height, frames,
                                          C.c_double(frame_interval), C.c_uint64(seed),
                                          C.c_void_p(out_ptr), device, C.c_void_p(stream)))


def run_device(frames_ptr: int, pixel_bytes: int, width: int, height: int, frames: int,
               out_ptr: int, precision: str = "f32", out_f64: bool = False, lags=None,
               q_max: Optional[float] = None, device: int = 0, stream: int = 0,
               timing: bool = True):
    """Device-resident WITH_FT (frames and map already in HBM, e.g. torch tensors' data_ptr).
    Returns (spatial_ms, temporal_ms, kernel_launches) of device time; timing=False keeps the
    call fully asynchronous (no host synchronisation) and returns zeros."""
    lag_arr = np.ascontiguousarray(np.asarray(lags if lags is not None else [], dtype=np.int64))
    sp, tp, nl = C.c_double(0), C.c_double(0), C.c_int(0)
    if not timing:
        _check(lib().ddm_b200_run_device(
            C.c_void_p(frames_ptr), pixel_bytes, width, height, frames,
            0 if precision == "f32" else 1, _p(lag_arr, C.c_int64) if len(lag_arr) else None,
            C.c_int64(len(lag_arr)), 0 if q_max is None else 1,
            C.c_double(0.0 if q_max is None else q_max), C.c_void_p(out_ptr), 1 if out_f64 else 0,
            device, C.c_void_p(stream), None, None, None))
        return 0.0, 0.0, 0
    _check(lib().ddm_b200_run_device(
        C.c_void_p(frames_ptr), pixel_bytes, width, height, frames,
        0 if precision == "f32" else 1, _p(lag_arr, C.c_int64) if len(lag_arr) else None,
        C.c_int64(len(lag_arr)), 0 if q_max is None else 1,
        C.c_double(0.0 if q_max is None else q_max), C.c_void_p(out_ptr), 1 if out_f64 else 0,
        device, C.c_void_p(stream), C.byref(sp), C.byref(tp), C.byref(nl)))
    return sp.value, tp.value, nl.value

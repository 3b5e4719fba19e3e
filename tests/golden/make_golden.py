"""Regenerate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (needs /root/reference and `make -C oracle`):
    python tests/golden/make_golden.py
Every array stored here was produced by the unmodified reference library
(oracle/_ref/libddmref.so = /root/reference/proj/core compiled with our FFTW-API shim).
Inputs are portable: the reference synth generator (mt19937_64 + Box-Muller,
`synth.cpp:98-132`) and u16 stacks drawn from mt19937_64 >> 48 (oracle.ddm_oracle.random_stack).
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import ddm_oracle as O  # noqa: E402
from oracle import ref  # noqa: E402

OUT = Path(__file__).resolve().parent

# (width, height, frames, seed, lags) — lags None = all
STACKS = [
    (8, 8, 16, 101, None),
    (16, 16, 64, 103, None),
    (25, 20, 30, 11, None),
    (1, 1, 5, 3, None),
    (3, 5, 7, 4, None),
    (6, 10, 12, 5, None),
    (32, 32, 100, 7, None),
    (50, 50, 100, 9, "log"),   # C5 analogue: non-power-of-two sizes (2 * 5^2)
    (64, 48, 200, 13, "log"),
]

SEQ_LENGTHS = [1, 2, 3, 5, 16, 100, 1000, 1024, 4096]


def seq_for(n: int, seed: int) -> np.ndarray:
    u = O.mt19937_64(seed, 2 * n).astype(np.float64) * 2.0 ** -64
    v = (2.0 * u - 1.0).reshape(n, 2)
    return v[:, 0] + 1j * v[:, 1]


def main() -> None:
    seqs = {}
    for n in SEQ_LENGTHS:
        s = seq_for(n, 40 + n)
        seqs[f"seq_{n}"] = s
        for prec in ("f64", "f32"):
            p = ref.with_ft_sequence(s, prec)
            seqs[f"d_{prec}_{n}"] = p.d
            seqs[f"da_{prec}_{n}"] = p.d_a
            seqs[f"corr_{prec}_{n}"] = p.corr
    np.savez_compressed(OUT / "sequences.npz", **seqs)

    stacks = {}
    for (w, h, n, seed, lagmode) in STACKS:
        key = f"{w}x{h}x{n}_s{seed}"
        st = O.random_stack(w, h, n, seed)
        lags = O.log_lags(n) if lagmode == "log" else []
        stacks[f"lags_{key}"] = np.asarray(lags if lags else range(n), dtype=np.int64)
        stacks[f"sha_{key}"] = np.frombuffer(hashlib.sha256(st.tobytes()).digest(), np.uint8)
        for prec in ("f64", "f32"):
            r = ref.run(st, "with_ft", prec, lags=lags, workers=4)
            stacks[f"map_{prec}_{key}"] = r.values
        if lagmode == "log":
            r = ref.run(st, "without_ft", "f64", lags=lags, workers=4)
            stacks[f"map_without_f64_{key}"] = r.values
    np.savez_compressed(OUT / "stacks.npz", **stacks)

    # C1 = configs[0] of BASELINE.json: 64x64 x 128 synthetic frames, reference synth seed 7
    st = ref.generate(64, 64, 128, particles=100, diffusion=0.5, seed=7)
    lags = O.log_lags(128)
    c1 = {"sha": np.frombuffer(hashlib.sha256(st.tobytes()).digest(), np.uint8),
          "lags": np.asarray(lags, dtype=np.int64),
          "first_frame": st[0]}
    for prec in ("f64", "f32"):
        r = ref.run(st, "with_ft", prec, lags=lags, workers=4)
        c1[f"map_{prec}"] = r.values
        c1[f"counters_{prec}"] = np.asarray([r.counters["spatial_ffts"],
                                             r.counters["temporal_ffts"]], dtype=np.int64)
    means, counts = ref.azimuthal_average(c1["map_f64"], lags, 64, 64)
    c1["radial_means_f64"] = means
    c1["radial_counts"] = counts
    np.savez_compressed(OUT / "c1_synth_seed7.npz", **c1)

    # synth generator goldens (bit-exact u16), a non-square, non-default parameter set
    syn = {}
    for (w, h, n, p, d, seed) in [(48, 40, 6, 30, 0.25, 3), (64, 64, 4, 100, 0.5, 7)]:
        syn[f"stack_{w}x{h}x{n}_p{p}_s{seed}"] = ref.generate(w, h, n, particles=p,
                                                              diffusion=d, seed=seed)
    np.savez_compressed(OUT / "synth.npz", **syn)

    pairwise()

    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)


def pairwise() -> None:
    """WITHOUT_FT and Direct maps + counters from the reference (pairwise.npz)."""
    out = {}
    for (w, h, n, seed, lagmode) in STACKS:
        key = f"{w}x{h}x{n}_s{seed}"
        st = O.random_stack(w, h, n, seed)
        lags = O.log_lags(n) if lagmode == "log" else []
        for prec in ("f64", "f32"):
            r = ref.run(st, "without_ft", prec, lags=lags, workers=4)
            out[f"without_{prec}_{key}"] = r.values
            out[f"without_{prec}_counters_{key}"] = np.asarray(
                [r.counters["spatial_ffts"], r.counters["temporal_ffts"], r.counters["pairs"]], np.int64)
        r = ref.run(st, "direct", "f32", lags=lags, workers=4)
        out[f"direct_{key}"] = r.values
        out[f"direct_counters_{key}"] = np.asarray(
            [r.counters["spatial_ffts"], r.counters["temporal_ffts"], r.counters["pairs"]], np.int64)
    # pass plan (`test_scheduler.cpp:182-197`): 16x16x64 seed 107 with budgets of 1 and 3 passes
    st = O.random_stack(16, 16, 64, 107)
    sb = 16 * 9 * 16
    for passes, cap in ((1, 64), (3, 22)):
        r = ref.run(st, "without_ft", "f64", memory_bytes=cap * sb, workers=2)
        out[f"passes{passes}_map"] = r.values
        out[f"passes{passes}_counters"] = np.asarray(
            [r.counters["spatial_ffts"], r.counters["temporal_ffts"], r.counters["pairs"]], np.int64)
        out[f"passes{passes}_budget"] = np.asarray([cap * sb], np.int64)
    # q_max cutoff + lag subset on without_ft
    st = O.random_stack(24, 20, 40, 211)
    r = ref.run(st, "without_ft", "f64", lags=[0, 1, 5, 39], q_max=6.5, workers=2)
    out["cut_map"] = r.values
    np.savez_compressed(OUT / "pairwise.npz", **out)


# `ddm analyze` cases: (name, format, W, H, N, seed, algorithm, precision, lags, q_max)
ANALYZE_CASES = [
    ("raw_f64_all", "raw_stack", 32, 24, 48, 31, "with_ft", "f64", (), None),
    ("pgm_f32_log_qmax", "pgm_dir", 24, 20, 40, 32, "with_ft", "f32", "log", 7.5),
    ("raw_f64_without", "raw_stack", 20, 16, 30, 33, "without_ft", "f64", (0, 1, 2, 3, 5, 8, 13), None),
    ("raw_f32_nofits", "raw_stack", 16, 16, 3, 34, "with_ft", "f32", (), None),
]


def write_stack(path: Path, fmt: str, st: np.ndarray, frame_interval: float = 0.25) -> None:
    """The inputs of ANALYZE_CASES: a raw stack (JSON header line + u16le) or a PGM directory
    (P5, maxval 65535, big-endian), the formats of `image_stack.cpp`."""
    n, h, w = st.shape
    if fmt == "raw_stack":
        with open(path, "wb") as f:
            f.write(json.dumps({"width": w, "height": h, "frames": n, "dtype": "u16le",
                                "frame_interval": frame_interval}).encode() + b"\n")
            f.write(st.astype("<u2").tobytes())
    else:
        path.mkdir(parents=True, exist_ok=True)
        for i, fr in enumerate(st):
            (path / f"f{i:05d}.pgm").write_bytes(f"P5\n{w} {h}\n65535\n".encode() + fr.astype(">u2").tobytes())


def analyze_case_stack(w, h, n, seed):
    return ref.generate(w, h, n, particles=30, diffusion=0.4, seed=seed)


def analyze() -> None:
    """Reference `ddm analyze` artefacts for ANALYZE_CASES -> tests/golden/analyze/<case>/."""
    import shutil
    import tempfile
    root = OUT / "analyze"
    shutil.rmtree(root, ignore_errors=True)
    for name, fmt, w, h, n, seed, alg, prec, lags, qm in ANALYZE_CASES:
        st = analyze_case_stack(w, h, n, seed)
        lag_list = O.log_lags(n) if lags == "log" else list(lags)
        with tempfile.TemporaryDirectory() as tmp:
            src = Path(tmp) / ("in" if fmt == "pgm_dir" else "in.raw")
            write_stack(src, fmt, st)
            ref.analyze(str(src), str(root / name), fmt, alg, prec, lag_list, qm, workers=2)
        print(name, sorted(p.name for p in (root / name).iterdir())[:4], "...")


# `ddm bench` sweep whose deterministic columns are pinned (budgets: ample, grouped, too small)
BENCH_SWEEP = dict(frame_counts=(16, 48), sizes=(16, 32), algorithms=("with_ft", "without_ft", "direct"),
                   workers=(2,), budgets=(1 << 30, 40000, 100))


def bench() -> None:
    """The reference's bench.csv for BENCH_SWEEP -> tests/golden/bench_sweep.csv (times are
    host-specific; the tests compare every other column)."""
    ref.bench_sweep(**BENCH_SWEEP, repetitions=1, warmup=0, out_csv=OUT / "bench_sweep.csv")
    print((OUT / "bench_sweep.csv").read_text())


if __name__ == "__main__":
    if sys.argv[1:] == ["pairwise"]:
        pairwise()
    elif sys.argv[1:] == ["analyze"]:
        analyze()
    elif sys.argv[1:] == ["bench"]:
        bench()
    else:
        main()

"""Pin the numpy oracle (oracle/ddm_oracle.py) to the reference.

Known-answer tests restate the reference's own unit tests
(`proj/tests/unit/test_temporal.cpp`, `test_spectrum.cpp`, `test_scheduler.cpp`) and the
golden fixtures in tests/golden/ were produced by the unmodified reference library
(tests/golden/make_golden.py).  CPU only.
"""
import hashlib
from pathlib import Path

import numpy as np
import pytest

from oracle import ddm_oracle as O

GOLD = Path(__file__).resolve().parent / "golden"


def rnd_seq(n, seed):
    r = np.random.default_rng(seed)
    return r.uniform(-1, 1, n) + 1j * r.uniform(-1, 1, n)


def test_pad_length_kats():  # test_temporal.cpp:36-58
    assert [O.pad_length(n) for n in (1, 2, 3, 100, 1000, 16384)] == [2, 4, 8, 256, 2048, 32768]
    prev = 0
    for n in range(1, 1025):
        p = O.pad_length(n)
        assert p >= 2 * n and p & (p - 1) == 0 and p >= prev and O.pad_length(2 * n) == 2 * p
        prev = p
    with pytest.raises(ValueError):
        O.pad_length(0)


def test_averages_and_correlation_kats():  # test_temporal.cpp:60-88
    ramp = np.array([[1, 2, 3]], dtype=np.complex128)
    np.testing.assert_allclose(O.averages_term(ramp)[0], [28 / 3, 9, 10], rtol=1e-14)
    np.testing.assert_allclose(O.correlation(ramp)[0], [14, 8, 3], rtol=1e-12)
    np.testing.assert_allclose(O.correlation(np.array([[1, -1]], dtype=complex))[0], [2, -1],
                               rtol=1e-12)


def test_with_ft_kats():  # test_temporal.cpp:90-118
    d = O.with_ft(np.array([[1, 2, 3]], dtype=complex))[0]
    assert abs(d[0]) < 1e-9 and d[1] == pytest.approx(1, rel=1e-12) and d[2] == pytest.approx(4, rel=1e-12)
    d = O.with_ft(np.array([[1, -1]], dtype=complex))[0]
    assert abs(d[0]) < 1e-9 and d[1] == pytest.approx(4, rel=1e-12)
    assert abs(O.with_ft(np.array([[3 + 4j]]))[0][0]) < 1e-9
    assert O.ramp_check()


@pytest.mark.parametrize("n", [1, 2, 3, 5, 16, 100])
def test_fft_path_matches_double_loop(n):  # test_temporal.cpp:120-132
    s = rnd_seq(n, 40 + n)[None]
    fast, slow = O.with_ft(s)[0], O.direct_sequence(s)[0]
    assert np.abs(fast - slow).max() <= 1e-9 * max(np.abs(slow).max(), 1.0)


def test_offset_and_scale_invariance():  # test_temporal.cpp:148-171
    s = rnd_seq(64, 11)[None]
    a, b = O.with_ft(s)[0], O.with_ft(s + (5 - 3j))[0]
    assert np.abs(a[1:] - b[1:]).max() <= 1e-9 * max(np.abs(a).max(), 1)
    s = rnd_seq(32, 13)[None]
    np.testing.assert_allclose(O.with_ft(2.5 * s)[0][1:], 6.25 * O.with_ft(s)[0][1:], rtol=1e-9)


def test_float_engine_near_double():  # test_temporal.cpp:200-211
    s = rnd_seq(64, 23)[None]
    a, b = O.with_ft(s, "f64")[0], O.with_ft(s.astype(np.complex64), "f32")[0]
    assert np.abs(a[1:] - b[1:]).max() <= 1e-4 * max(np.abs(a).max(), 1)


def test_oracle_matches_reference_sequences():
    g = np.load(GOLD / "sequences.npz")
    for n in (1, 2, 3, 5, 16, 100, 1000, 1024, 4096):
        s = g[f"seq_{n}"][None]
        for prec, tol in (("f64", 1e-12), ("f32", 2e-5)):
            d = O.with_ft(s.astype(np.complex64) if prec == "f32" else s, prec)[0]
            ref = g[f"d_{prec}_{n}"]
            scale = max(np.abs(ref).max(), 1.0)
            assert np.abs(d - ref).max() <= tol * scale, (n, prec)


def _stack_keys():
    g = np.load(GOLD / "stacks.npz")
    return sorted(k[len("lags_"):] for k in g.files if k.startswith("lags_"))


@pytest.mark.parametrize("key", _stack_keys())
def test_oracle_matches_reference_maps(key):
    g = np.load(GOLD / "stacks.npz")
    dims, seed = key.split("_s")
    w, h, n = map(int, dims.split("x"))
    st = O.random_stack(w, h, n, int(seed))
    assert hashlib.sha256(st.tobytes()).digest() == g[f"sha_{key}"].tobytes()
    lags = g[f"lags_{key}"]
    for prec, tol in (("f64", 1e-12), ("f32", 1e-5)):
        m = O.run_with_ft(st, prec, lags=lags)
        ref = g[f"map_{prec}_{key}"]
        assert O.relative_deviation(m, ref) <= tol, (key, prec)
        assert O.relative_l2(m, ref) <= tol
    if f"map_without_f64_{key}" in g.files:  # three-way agreement (acceptance_main.cpp:126-150)
        ref_wo = g[f"map_without_f64_{key}"]
        assert O.relative_deviation(O.run_without_ft(st, "f64", lags=lags), ref_wo) <= 1e-12
        assert O.relative_deviation(g[f"map_f64_{key}"], ref_wo) <= 1e-9


def test_c1_golden_and_radial():
    g = np.load(GOLD / "c1_synth_seed7.npz")
    lags = g["lags"]
    # map of the reference f64 run vs f32 run of the same frames: the f32 budget
    assert O.relative_l2(g["map_f32"], g["map_f64"]) < 1e-5
    means, counts = O.azimuthal_average(g["map_f64"], 64, 64)
    np.testing.assert_array_equal(counts, g["radial_counts"])
    np.testing.assert_allclose(means, g["radial_means_f64"], rtol=1e-12, atol=1e-9)
    assert list(g["counters_f64"]) == [128, 2 * 64 * 33]


def test_geometry():  # test_spectrum.cpp:130-188
    assert O.cutoff_set(512, 512).size == 512 * 257
    assert O.cutoff_set(8, 8, 0.0).tolist() == [0]
    assert float(O.q_magnitude(7, 0, 8)) == pytest.approx(1.0)
    assert float(O.q_magnitude(4, 0, 8)) == pytest.approx(4.0)
    assert float(O.q_magnitude(5, 2, 8)) == pytest.approx(np.sqrt(13.0))
    np.testing.assert_array_equal(O.cutoff_set(8, 4), np.arange(20))


def test_planner_arithmetic():  # test_scheduler.cpp:58-71
    cap, groups = O.plan_with_ft(131584, 16384, 23 << 30, "f64")
    assert cap == 94208 and groups == [(0, 94208), (94208, 131584)]
    cap, groups = O.plan_with_ft(131584, 16384, 8 << 30, "f64")
    assert cap == 32768 and len(groups) == 5
    with pytest.raises(MemoryError):
        O.plan_with_ft(10, 1024, 1024, "f64")


def test_oracle_against_live_reference():
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    st = O.random_stack(12, 10, 40, 77)
    for prec in ("f64", "f32"):
        r = ref.run(st, "with_ft", prec, workers=3)
        assert O.relative_deviation(O.run_with_ft(st, prec), r.values) <= (1e-12 if prec == "f64" else 1e-5)
        assert r.counters["temporal_ffts"] == 2 * 10 * 7


def test_pairwise_goldens_pin_the_oracle():
    """WITHOUT_FT / Direct maps produced by the reference (tests/golden/pairwise.npz) against
    the numpy restatement (`pairwise.cpp:11-116`)."""
    g = np.load(GOLD / "pairwise.npz")
    for (w, h, n, seed, lagmode) in [(8, 8, 16, 101, None), (25, 20, 30, 11, None),
                                     (50, 50, 100, 9, "log")]:
        key = f"{w}x{h}x{n}_s{seed}"
        st = O.random_stack(w, h, n, seed)
        lags = O.log_lags(n) if lagmode == "log" else None
        ref = g[f"without_f64_{key}"]
        assert O.relative_deviation(O.run_without_ft(st, "f64", lags=lags), ref) <= 1e-12
        # Eq. 1 equals the spectral differences (linearity of the transform)
        assert O.relative_deviation(g[f"direct_{key}"], ref) <= 1e-9
        pairs = sum(n - m for m in O.normalize_lags(lags, n) if m > 0)
        assert g[f"direct_counters_{key}"][2] == pairs


def test_fit_restatement_recovers_a_known_relaxation():
    t = np.arange(1, 200, dtype=np.float64) * 0.5
    y = 3.0 * (1.0 - np.exp(-t / 7.5)) + 0.25
    a, b, tau, res, flag = O.fit_exponential(t, y)
    assert flag == "ok" and abs(tau - 7.5) < 1e-6 and abs(a - 3.0) < 1e-6 and abs(b - 0.25) < 1e-6
    assert O.fit_exponential(t, np.full_like(t, 2.0))[4] == "degenerate"
    d, used = O.estimate_diffusion({2: (1, 0, 1 / (0.3 * (2 * np.pi * 2 / 64) ** 2), 0, "ok"),
                                    3: (1, 0, 1 / (0.3 * (2 * np.pi * 3 / 64) ** 2), 0, "ok")}, 64, 2, 10)
    assert used == 2 and abs(d - 0.3) < 1e-12


def test_estimate_diffusion_through_the_abi():
    """Host-only C-ABI entry (no device): the same least squares as the oracle."""
    from paper_2012_05695_b200 import ddm
    if not ddm.LIB_PATH.exists():
        pytest.skip("library not built")
    taus = np.array([0, 0, 1 / (0.3 * (2 * np.pi * 2 / 64) ** 2), 5.0, 1 / (0.3 * (2 * np.pi * 4 / 64) ** 2)])
    flags = np.array([-1, 0, 0, 2, 0], dtype=np.int32)
    d, used = ddm.estimate_diffusion(taus, flags, 64, 2, 10)
    assert used == 2 and abs(d - 0.3) < 1e-12


# ------------------------------------------------------- `ddm analyze` artefacts (goldens)

ANALYZE_GOLD = Path(__file__).resolve().parent / "golden" / "analyze"


@pytest.mark.parametrize("case", sorted(p.name for p in ANALYZE_GOLD.iterdir()))
def test_analyze_golden_restated(case):
    """The reference's radial.csv / fits.csv (tests/golden/analyze, written by the reference
    library via oracle/ref_capi.cpp:ref_analyze) follow from its own d_m*.bin maps under the
    oracle's azimuthal_average and fit_exponential restatements."""
    from golden.artifacts import read_artifacts
    a = read_artifacts(ANALYZE_GOLD / case)
    idx = a["index"]
    lags = sorted(a["maps"])
    assert lags == idx["lags"]
    vals = np.stack([a["maps"][m] for m in lags])
    means, counts = O.azimuthal_average(vals, idx["width"], idx["height"], idx["q_max"])
    expect = [(m, b) for m in lags for b in range(len(counts)) if counts[b] > 0]
    assert [(r[0], r[1]) for r in a["radial"]] == expect
    for (m, b, mean, cnt) in a["radial"]:
        assert cnt == counts[b]
        assert abs(mean - means[lags.index(m), b]) <= 1e-12 * max(abs(mean), 1e-300)
    usable = [i for i, m in enumerate(lags) if m >= 1]
    if len(usable) < 4:
        assert a["fits"] is None
        return
    t = np.asarray([lags[i] for i in usable], float) * idx["frame_interval"]
    fitted = [b for b in range(len(counts)) if counts[b] > 0]
    assert [r[0] for r in a["fits"]] == fitted
    for (b, A, B, tau, res, flag) in a["fits"]:
        oA, oB, otau, ores, oflag = O.fit_exponential(t, means[usable, b], idx["frame_interval"])
        assert oflag == flag, (b, flag, oflag)
        if flag == "ok":
            assert abs(otau - tau) <= 1e-6 * tau and abs(ores - res) <= 1e-6 * max(res, 1e-300)

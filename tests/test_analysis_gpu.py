"""The reference's analysis unit tests (`proj/tests/unit/test_analysis.cpp`) and pairwise
unit tests (`test_pairwise.cpp`), restated against the device implementations: the ring
average (`radial_kernel`), the ring fits (`fit_rings_kernel`), the diffusion estimate and the
WITHOUT_FT / Direct engines. GPU only (the CPU-side oracle checks live in test_oracle.py)."""
import numpy as np
import pytest

from oracle import ddm_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ddm():
    from paper_2012_05695_b200 import ddm as m
    if m.device_count() < 1:
        pytest.skip("no CUDA device")
    return m


def _profile(a, b, tau, dt, n_lags):
    """model_profile of test_analysis.cpp: one bin, lags 0..n-1, d = a (1 - e^{-t/tau}) + b."""
    lags = np.arange(n_lags, dtype=np.int64)
    t = lags * dt
    means = (a * (1.0 - np.exp(-t / tau)) + b).reshape(n_lags, 1)
    means[0] = 0.0
    return means, lags, np.array([1], dtype=np.int64)


# ----------------------------------------------------------------------- ring average

def test_constant_map_averages_to_itself(ddm):
    vals = np.full((3, 8, 5), 5.25)
    means, counts = ddm.azimuthal_average(vals, 8, 8)
    assert counts.sum() == 8 * 5
    assert np.all(np.abs(means[:, counts > 0] - 5.25) <= 5.25e-14)


def test_radius_valued_map_recovers_its_bin(ddm):
    flat = O.cutoff_set(8, 8)
    q = O.q_magnitude(flat // 5, flat % 5, 8)
    vals = np.zeros((1, 8 * 5))
    vals[0, flat] = q
    means, counts = ddm.azimuthal_average(vals.reshape(1, 8, 5), 8, 8)
    for b in np.nonzero(counts)[0]:
        assert abs(means[0, b] - b) <= 0.5


def test_zero_cutoff_collapses_to_dc(ddm):
    vals = np.zeros((1, 8, 5))
    vals[0, 0, 0] = 42.0
    means, counts = ddm.azimuthal_average(vals, 8, 8, q_max=0.0)
    assert means.shape[1] == 1 and counts[0] == 1 and means[0, 0] == 42.0


def test_averaging_commutes_with_scaling(ddm):
    rng = np.random.default_rng(7)
    vals = rng.uniform(0.0, 10.0, (2, 16, 9))
    m1, _ = ddm.azimuthal_average(vals, 16, 16)
    m2, _ = ddm.azimuthal_average(2.0 * vals, 16, 16)
    np.testing.assert_allclose(m2, 2.0 * m1, rtol=1e-12)


# ----------------------------------------------------------------------- fits

def test_exact_exponential_is_recovered(ddm):
    means, lags, counts = _profile(2.0, 0.5, 5.0, 0.5, 64)
    a, b, tau, res, flag = ddm.fit_rings(means, lags, counts, 0.5)
    assert flag[0] == 0
    assert abs(a[0] - 2.0) <= 2e-6 and abs(b[0] - 0.5) <= 5e-6 and abs(tau[0] - 5.0) <= 5e-6
    assert res[0] <= 1e-8


@pytest.mark.parametrize("tau0", [0.8, 3.0, 40.0])
def test_slow_and_fast_relaxations_converge(ddm, tau0):
    means, lags, counts = _profile(1.5, 0.1, tau0, 1.0, 128)
    _, _, tau, _, flag = ddm.fit_rings(means, lags, counts, 1.0)
    assert flag[0] == 0 and abs(tau[0] - tau0) <= 1e-4 * tau0


def test_flat_data_is_degenerate(ddm):
    means, lags, counts = _profile(0.0, 3.0, 5.0, 1.0, 32)
    means[0] = 3.0
    a, b, tau, _, flag = ddm.fit_rings(means, lags, counts, 1.0)
    assert flag[0] == 1 and a[0] == 0.0 and tau[0] > 0.0


def test_mild_noise_does_not_derail_the_fit(ddm):
    means, lags, counts = _profile(2.0, 0.5, 8.0, 1.0, 128)
    means[1:, 0] += np.random.default_rng(11).normal(0.0, 0.02, 127)
    _, _, tau, _, flag = ddm.fit_rings(means, lags, counts, 1.0)
    assert flag[0] == 0 and abs(tau[0] - 8.0) <= 0.05 * 8.0


def test_too_few_lags_are_not_fitted(ddm):
    means, lags, counts = _profile(1.0, 0.0, 2.0, 1.0, 3)
    assert ddm.fit_rings(means, lags, counts, 1.0)[4][0] == -1


def test_fit_all_bins_skips_empty_bins(ddm):
    lags = np.arange(64, dtype=np.int64)
    t = lags.astype(float)
    means = np.zeros((64, 3))
    means[:, 0] = 2.0 * (1.0 - np.exp(-t / 4.0))
    means[:, 2] = 1.0 * (1.0 - np.exp(-t / 9.0))
    _, _, tau, _, flag = ddm.fit_rings(means, lags, np.array([4, 0, 2]), 1.0)
    assert list(flag) == [0, -1, 0]
    assert abs(tau[0] - 4.0) <= 4e-4 and abs(tau[2] - 9.0) <= 9e-4


def test_diffusion_slope_from_ideal_rates(ddm):
    bins = np.arange(13)
    tau = np.zeros(13)
    tau[1:] = 1.0 / (0.7 * (2 * np.pi * bins[1:] / 64.0) ** 2)
    flag = np.zeros(13, dtype=np.int32)
    flag[0] = -1
    d, used = ddm.estimate_diffusion(tau, flag, 64, 2, 10)
    assert used == 9 and abs(d - 0.7) <= 0.7e-12
    flag[4] = 1
    d, used = ddm.estimate_diffusion(tau, flag, 64, 2, 10)
    assert used == 8 and abs(d - 0.7) <= 0.7e-12


# ----------------------------------------------------------------------- pairwise

def _cfg(ddm, alg, **kw):
    kw.setdefault("memory_bytes", 1 << 40)
    return ddm.RunConfig(algorithm=alg, **kw)


def test_identical_frames_difference_to_zero(ddm):
    st = np.repeat(O.random_stack(12, 10, 1, seed=3), 6, axis=0)
    for alg in ("without_ft", "direct"):
        assert np.all(ddm.run(st, _cfg(ddm, alg, precision="f64")).values == 0.0)


def test_single_pixel_stack_is_the_scalar_sequence(ddm):
    st = O.random_stack(1, 1, 40, seed=9)
    a = ddm.run(st, _cfg(ddm, "without_ft", precision="f64")).values.reshape(40)
    s = st.reshape(40).astype(np.float64)
    ref = [0.0] + [np.mean((s[m:] - s[:-m]) ** 2) for m in range(1, 40)]
    np.testing.assert_allclose(a, ref, rtol=1e-13)


def test_lag_beyond_the_stack_throws(ddm):
    st = O.random_stack(8, 8, 5, seed=2)
    with pytest.raises(ddm.InputError):
        ddm.run(st, _cfg(ddm, "without_ft", precision="f64", lags=[0, 5]))


def test_lag_zero_plane_and_sparse_pair_count(ddm):
    st = O.random_stack(8, 6, 30, seed=4)
    a = ddm.run(st, _cfg(ddm, "without_ft", precision="f64", lags=[0, 3, 17]))
    assert np.all(a.values[0] == 0.0)
    assert a.counters["pairs"] == (30 - 3) + (30 - 17)
    b = ddm.run(O.random_stack(16, 16, 30, seed=4), _cfg(ddm, "without_ft", precision="f64", lags=[3, 17]))
    assert b.counters["pairs"] == a.counters["pairs"]   # independent of the wave-vector count


def test_cutoff_coefficients_stay_zero(ddm):
    st = O.random_stack(16, 12, 20, seed=8)
    a = ddm.run(st, _cfg(ddm, "without_ft", precision="f64", q_max=3.0)).values
    keep = np.zeros(12 * 9, bool)
    keep[O.cutoff_set(16, 12, 3.0)] = True
    assert np.all(a.reshape(20, -1)[:, ~keep] == 0.0)
    assert np.any(a.reshape(20, -1)[1:, keep] != 0.0)


def test_float_spectra_within_single_precision(ddm):
    st = O.random_stack(16, 16, 48, seed=12)
    a = ddm.run(st, _cfg(ddm, "without_ft", precision="f32")).values
    b = ddm.run(st, _cfg(ddm, "without_ft", precision="f64")).values
    assert O.relative_deviation(a, b) <= 1e-5

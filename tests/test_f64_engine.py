"""The f64 warp temporal engine (temporal_warp64.cu, N2 = 2048) and the f64 register spatial
kernels against the numpy oracle at the f64 bound (relative L2 <= 1e-10, `BASELINE.json`):
FULL (N = 1024) and runtime-N (N = 600, 1000) variants, register and generic spatial passes,
lag lists, a cutoff, the group / partial path and the engine report."""
import numpy as np
import pytest

from oracle import ddm_oracle as O

pytestmark = pytest.mark.gpu
F64_L2 = 1e-10


@pytest.fixture(scope="module")
def ddm():
    from paper_2012_05695_b200 import ddm
    if ddm.device_count() < 1:
        pytest.skip("no CUDA device")
    return ddm


@pytest.mark.parametrize("W,H,N,spatial", [
    (64, 64, 1024, "rows2<32>"),     # FULL, register spatial in f64
    (48, 40, 600, "generic"),        # runtime N, generic spatial (q-major, T = 1)
    (32, 64, 1000, "rows2<16>"),     # runtime N, register spatial
])
def test_f64_engine_vs_oracle(ddm, W, H, N, spatial):
    st = O.random_stack(W, H, N, seed=N + W)
    a = ddm.run(st, ddm.RunConfig(precision="f64", memory_bytes=1 << 40))
    eng = ddm.last_engines()
    assert "warp64<1024>" in eng and spatial in eng, eng
    ref = O.run_with_ft(st, "f64")
    assert O.relative_l2(a.values, ref) <= F64_L2
    assert np.all(a.values[0] == 0.0)


def test_f64_engine_lags_cutoff_and_groups(ddm):
    st = O.random_stack(64, 32, 800, seed=9)
    full = O.run_with_ft(st, "f64")
    lags = [0, 1, 7, 100, 799]
    a = ddm.run(st, ddm.RunConfig(precision="f64", lags=lags, memory_bytes=1 << 40))
    assert "warp64<1024>" in ddm.last_engines()
    assert O.relative_l2(a.values, full[lags]) <= F64_L2
    # cutoff: zeros outside, the oracle inside
    c = ddm.run(st, ddm.RunConfig(precision="f64", q_max=7.5, memory_bytes=1 << 40))
    flat = ddm.cutoff_set(64, 32, 7.5)
    got = c.values.reshape(c.values.shape[0], -1)
    mask = np.zeros(got.shape[1], bool)
    mask[flat] = True
    assert np.all(got[:, ~mask] == 0.0)
    assert O.relative_l2(got[:, mask], full.reshape(full.shape[0], -1)[:, mask]) <= F64_L2
    # several groups (partial files, the reference's group semantics): same map
    g = ddm.run(st, ddm.RunConfig(precision="f64", memory_bytes=64 * 32 * 16 * 800 // 3))
    assert g.counters["spatial_ffts"] > 800
    assert O.relative_l2(g.values, full) <= F64_L2

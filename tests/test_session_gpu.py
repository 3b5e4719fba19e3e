"""Opaque staging session of the C-ABI (`ddm_b200_create` / `_stage_frames` / `_run_with_ft`,
SURVEY.md §8b): stage once, run several requests, each equal to `ddm::run`'s WithFt branch
(`scheduler.cpp:413-483`) on the same frames: the full map bitwise, wave-vector lists against
the cutoff run of the same list, lag lists, counters, errors, and two sessions on one GPU at
once from two threads."""
import threading

import numpy as np
import pytest

from oracle import ddm_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ddm():
    from paper_2012_05695_b200 import ddm
    if ddm.device_count() < 1:
        pytest.skip("no CUDA device")
    return ddm


def test_session_equals_run_and_serves_several_requests(ddm):
    st = ddm.generate(64, 64, 1024, particles=100, diffusion=0.5, seed=11)
    ref = ddm.run(st, ddm.RunConfig(precision="f32", memory_bytes=1 << 40))
    with ddm.Session(64, 64, 1024, "f32") as s:
        s.stage(st[:300], 0)           # staged in pieces, out of order
        s.stage(st[700:], 700)
        s.stage(st[300:700], 300)
        got, counters, timing = s.run_with_ft()
        assert "warp<1024>" in s.engines() and "rows2<32>" in s.engines()
        assert np.array_equal(got, ref.values)          # same kernels, bitwise
        assert counters == {"spatial_ffts": 1024, "temporal_ffts": 2 * 64 * 33, "pairs": 0}
        assert timing["total"] > 0
        # lag subset (unsorted: normalised like RunConfig::lags, `result_map.cpp` normalize_lags)
        sub, _, _ = s.run_with_ft(lags=[5, 1, 1000, 0])
        assert np.array_equal(sub, ref.values[[0, 1, 5, 1000]])
        with pytest.raises(ddm.InputError, match="duplicate"):
            s.run_with_ft(lags=[5, 5])
        # a wave-vector list: the cutoff run of the same list
        cut = ddm.run(st, ddm.RunConfig(precision="f32", q_max=9.5, memory_bytes=1 << 40))
        flat = ddm.cutoff_set(64, 64, 9.5)
        part, c2, _ = s.run_with_ft(wave_vectors=flat)
        assert np.array_equal(part, cut.values)
        assert c2["temporal_ffts"] == 2 * len(flat)
        mask = np.zeros(64 * 33, bool)
        mask[flat] = True
        assert np.all(part.reshape(part.shape[0], -1)[:, ~mask] == 0.0)


def test_session_f64_against_the_oracle(ddm):
    st = O.random_stack(48, 40, 96, seed=5)
    with ddm.Session(48, 40, 96, "f64") as s:
        s.stage(st)
        got, _, _ = s.run_with_ft()
    ref = O.run_with_ft(st, "f64")
    assert O.relative_l2(got, ref) <= 1e-10
    assert np.all(got[0] == 0.0)


def test_session_u8_frames(ddm):
    st8 = (O.random_stack(32, 32, 64, seed=3) % 256).astype(np.uint8)
    with ddm.Session(32, 32, 64, "f32") as s:
        s.stage(st8)
        got, _, _ = s.run_with_ft()
        with pytest.raises(ddm.InputError):
            s.stage(st8[:1].astype(np.uint16), 0)      # a session is all u8 or all u16
    ref = ddm.run(st8.astype(np.uint16), ddm.RunConfig(precision="f32", memory_bytes=1 << 40))
    assert np.array_equal(got, ref.values)


def test_session_errors(ddm):
    with pytest.raises(ddm.InputError):
        ddm.Session(0, 32, 64)
    with pytest.raises(ddm.InputError):
        ddm.Session(32, 32, 64, device=99)
    st = O.random_stack(32, 32, 64, seed=2)
    with ddm.Session(32, 32, 64) as s:
        s.stage(st[:10])
        with pytest.raises(ddm.InputError, match="staged"):
            s.run_with_ft()
        with pytest.raises(ddm.InputError):
            s.stage(st[:10], 60)                        # beyond the stack
        s.stage(st[10:], 10)
        with pytest.raises(ddm.InputError):
            s.run_with_ft(wave_vectors=[5, 3])          # not ascending
        with pytest.raises(ddm.InputError):
            s.run_with_ft(wave_vectors=[32 * 17])       # outside the plane
        with pytest.raises(ddm.InputError):
            s.run_with_ft(lags=[64])                    # lag >= frames
        got, _, _ = s.run_with_ft(lags=[0, 63])
        assert got.shape == (2, 32, 17)


def test_two_sessions_concurrently(ddm):
    a = ddm.generate(64, 64, 600, particles=50, diffusion=0.4, seed=1)
    b = ddm.generate(64, 64, 600, particles=50, diffusion=0.9, seed=2)
    want = [ddm.run(x, ddm.RunConfig(precision="f32", memory_bytes=1 << 40)).values for x in (a, b)]
    out = [None, None]

    def work(i, st):
        with ddm.Session(64, 64, 600, "f32") as s:
            s.stage(st)
            for _ in range(3):
                out[i], _, _ = s.run_with_ft()

    ts = [threading.Thread(target=work, args=(i, x)) for i, x in enumerate((a, b))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert np.array_equal(out[0], want[0]) and np.array_equal(out[1], want[1])

"""Host-side logic of the library calls that needs no device: `ddm bench` sweep validation
(`bench.cpp:95-117`) and `ddm analyze` input errors, raised before any CUDA work."""
import pytest

from paper_2012_05695_b200 import ddm


@pytest.mark.parametrize("kw, msg", [
    (dict(frame_counts=(), sizes=(16,)), "every axis"),
    (dict(frame_counts=(0,), sizes=(16,)), "frame count 0"),
    (dict(frame_counts=(70000,), sizes=(16,)), "frame count 70000"),
    (dict(frame_counts=(16,), sizes=(2048,)), "size 2048"),
    (dict(frame_counts=(16,), sizes=(16,), workers=(0,)), "worker count"),
    (dict(frame_counts=(16,), sizes=(16,), budgets=(0,)), "budget must be positive"),
    (dict(frame_counts=(16,), sizes=(16,), repetitions=0), "repetitions"),
    (dict(frame_counts=(16,), sizes=(16,), warmup=-1), "warmup"),
])
def test_bench_sweep_validation(tmp_path, kw, msg):
    with pytest.raises(ddm.InputError, match=msg):
        ddm.bench_sweep(out=str(tmp_path), **kw)


def test_bench_sweep_unknown_algorithm(tmp_path):
    with pytest.raises(ddm.InputError):
        ddm.bench_sweep((16,), (16,), algorithms=("fastest",), out=str(tmp_path))


def test_analyze_missing_input_is_io_error(tmp_path):
    with pytest.raises(ddm.IoError):
        ddm.analyze(str(tmp_path / "none.raw"), str(tmp_path / "o"), ddm.RunConfig(), fmt="raw_stack")
    with pytest.raises(ddm.InputError):
        ddm.analyze(str(tmp_path), str(tmp_path / "o"), ddm.RunConfig(), fmt="tiff")

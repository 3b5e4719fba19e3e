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


def test_synth_writes_the_generated_stack_and_manifest(tmp_path):
    """`ddm synth` (`ddm_cli.cpp:306-327`): stack.raw holds ddm::generate's frames (bit-identical
    to the reference generator, tests/golden/synth.npz pins that) behind the raw-stack header;
    synth.json echoes every SynthConfig field (`synth.cpp:134-155`)."""
    import json
    import numpy as np
    path = ddm.synth(str(tmp_path / "s"), size=24, frames=10, particles=7, diffusion=0.3,
                     frame_interval=0.5, seed=11)
    st = ddm.load_stack(path, "raw_stack")
    assert np.array_equal(st, ddm.generate(24, 24, 10, particles=7, diffusion=0.3, frame_interval=0.5, seed=11))
    with open(path, "rb") as f:
        hdr = json.loads(f.readline())
    assert hdr == {"width": 24, "height": 24, "frames": 10, "dtype": "u16le", "frame_interval": 0.5}
    man = json.loads((tmp_path / "s" / "synth.json").read_text())
    assert man == {"tool_version": "0.1.0-b200", "generator": "mt19937_64/box-muller", "particles": 7,
                   "diffusion": 0.3, "psf_sigma": 1.0, "amplitude": 1000.0, "background": 100.0,
                   "width": 24, "height": 24, "frames": 10, "frame_interval": 0.5, "seed": 11}


def test_synth_rejects_bad_config(tmp_path):
    with pytest.raises(ddm.InputError):
        ddm.synth(str(tmp_path / "s"), size=0)


def test_compare_needs_two_known_algorithms(tmp_path):
    with pytest.raises(ddm.InputError):
        ddm.compare("x.raw", ddm.RunConfig(), algorithms=("with_ft",))
    with pytest.raises(ddm.InputError):
        ddm.compare("x.raw", ddm.RunConfig(), algorithms=("with_ft", "fast"))


def test_crossover_reports_the_first_frame_count_that_wins():
    """`test_bench.cpp:109-128`: N* is the first N whose with_ft total beats without_ft's;
    a size where it never does reports none; sizes in first-seen order."""
    cells = [("with_ft", 256, 32, 5.0), ("without_ft", 256, 32, 1.0),
             ("with_ft", 512, 32, 3.0), ("without_ft", 512, 32, 2.5),
             ("with_ft", 1024, 32, 2.0), ("without_ft", 1024, 32, 4.0),
             ("with_ft", 256, 64, 9.0), ("without_ft", 256, 64, 1.0)]
    assert list(ddm.crossover(cells).items()) == [(32, 1024), (64, None)]


def test_crossover_skips_failed_cells():
    """Failed cells (a plan that did not fit) never win or lose (`bench.cpp:158-166`)."""
    cells = [("with_ft", 64, 16, 1.0, True), ("without_ft", 64, 16, 2.0),
             ("with_ft", 128, 16, 1.0), ("without_ft", 128, 16, 2.0)]
    assert ddm.crossover(cells) == {16: 128}
    assert ddm.crossover([]) == {}

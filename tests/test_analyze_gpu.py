"""`ddm analyze` as a library call (§8f rank 1): ddm_b200_analyze writes the reference CLI's
artefact set (`proj/tools/ddm_cli.cpp:206-240`) — d_m<lag>.bin + index.json (write_results,
`archive.cpp:60-110`), radial.csv and fits.csv (`analysis.cpp:273-304`) — and the files are
compared with the reference library's own output for the same input (tests/golden/analyze,
written by `make_golden.py analyze` through oracle/ref_capi.cpp:ref_analyze).

Tolerances: maps and ring means 1e-10 relative for f64, relative L2 1e-4 for f32 (north
star); integer fields (lags, bins, counts, counters, manifest) exact; fits: same rings and
flags, ok-fit parameters within 1e-6 (f64 maps) / 1e-3 (f32 maps) relative — the device
LM sums in warp-tree order, the reference sequentially.
"""
import json
from pathlib import Path

import numpy as np
import pytest

from golden.artifacts import read_artifacts, stable_index
from golden.make_golden import ANALYZE_CASES, write_stack
from oracle import ddm_oracle as O

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden" / "analyze"


@pytest.fixture(scope="module")
def ddm():
    from paper_2012_05695_b200 import ddm as D
    if D.device_count() < 1:
        pytest.skip("no CUDA device")
    return D


def _analyze(ddm, tmp_path, case):
    name, fmt, w, h, n, seed, alg, prec, lags, qm = case
    st = ddm.generate(w, h, n, particles=30, diffusion=0.4, seed=seed)
    src = tmp_path / ("in" if fmt == "pgm_dir" else "in.raw")
    write_stack(src, fmt, st)
    lag_list = O.log_lags(n) if lags == "log" else list(lags)
    cfg = ddm.RunConfig(algorithm=alg, precision=prec, lags=lag_list, q_max=qm,
                        memory_bytes=1 << 40, workers=2)
    out = tmp_path / "out"
    info = ddm.analyze(str(src), str(out), cfg, fmt="auto")
    return info, read_artifacts(out), read_artifacts(GOLD / name)


@pytest.mark.parametrize("case", ANALYZE_CASES, ids=[c[0] for c in ANALYZE_CASES])
def test_analyze_artifacts_match_reference(ddm, tmp_path, case):
    prec_f64 = case[7] == "f64"
    info, got, ref = _analyze(ddm, tmp_path, case)
    assert got["files"] == sorted(ref["files"] + ["run.json"])
    # the workspace is out_dir, so the group partials stay beside the maps (scheduler.cpp:447)
    ls = lambda d: sorted(p.name for p in (d / "partials").iterdir()) if (d / "partials").is_dir() else []  # noqa: E731,E501
    assert ls(tmp_path / "out") == ls(GOLD / case[0])
    assert stable_index(got["index"]) == stable_index(ref["index"])
    assert info["n_lags"] == len(ref["index"]["lags"])
    assert info["fits_written"] == (ref["fits"] is not None)
    for m, r in ref["maps"].items():
        g = got["maps"][m]
        if prec_f64:
            assert O.relative_deviation(g, r) <= 1e-10, m
        else:
            assert O.relative_l2(g, r) <= 1e-4, m
    assert [x[:2] + x[3:] for x in got["radial"]] == [x[:2] + x[3:] for x in ref["radial"]]
    g = np.asarray([x[2] for x in got["radial"]])
    r = np.asarray([x[2] for x in ref["radial"]])
    if prec_f64:
        assert O.relative_deviation(g, r) <= 1e-10
    else:
        assert O.relative_l2(g, r) <= 1e-4
    if ref["fits"] is None:
        assert got["fits"] is None
        return
    assert [(x[0], x[5]) for x in got["fits"]] == [(x[0], x[5]) for x in ref["fits"]]
    tol = 1e-6 if prec_f64 else 1e-3
    for gf, rf in zip(got["fits"], ref["fits"]):
        if rf[5] != "ok":
            continue
        scale = max(abs(rf[1]), abs(rf[2]))
        assert abs(gf[1] - rf[1]) <= tol * scale and abs(gf[2] - rf[2]) <= tol * scale, gf
        assert abs(gf[3] - rf[3]) <= tol * rf[3], (gf, rf)


def test_analyze_run_json_echo(ddm, tmp_path):
    """The CLI's option echo (`ddm_cli.cpp:189-203`, `:226-229`) beside the artefacts."""
    case = ANALYZE_CASES[0]
    _analyze(ddm, tmp_path, case)
    echo = json.loads((tmp_path / "out" / "run.json").read_text())
    assert echo["subcommand"] == "analyze" and echo["algorithm"] == "with_ft"
    assert echo["format"] == "raw_stack" and echo["precision"] == "f64"
    assert set(echo) == {"tool_version", "input", "format", "lags", "q_max", "memory_limit_bytes",
                         "workers", "precision", "out", "subcommand", "algorithm"}


def test_analyze_rejects_missing_input(ddm, tmp_path):
    with pytest.raises(ddm.IoError):
        ddm.analyze(str(tmp_path / "nope.raw"), str(tmp_path / "o"), ddm.RunConfig(), fmt="raw_stack")


# ----------------------------------------------------------------- `ddm bench` sweep

def test_bench_sweep_matches_reference_columns(ddm, tmp_path):
    """Every deterministic column of bench.csv (cells, planned groups/passes, counters,
    failed rows) equals the reference sweep's (tests/golden/bench_sweep.csv, written by
    `make_golden.py bench` through the reference's own ddm::sweep); the crossover is the
    first N whose with_ft median total beats without_ft's (`bench.cpp:144-183`)."""
    import csv
    from golden.make_golden import BENCH_SWEEP
    rows, xo = ddm.bench_sweep(**BENCH_SWEEP, repetitions=2, warmup=1, out=str(tmp_path))
    with open(GOLD.parent / "bench_sweep.csv", newline="") as f:
        ref_rows = list(csv.DictReader(f))
    timed = {"seconds_total", "seconds_disk", "seconds_step1", "seconds_step2", "seconds_merge"}
    assert len(rows) == len(ref_rows)
    for g, r in zip(rows, ref_rows):
        assert {k: v for k, v in g.items() if k not in timed} == {k: v for k, v in r.items() if k not in timed}
        if r["seconds_total"] == "nan":
            assert all(g[k] == "nan" for k in timed)
        else:
            assert float(g["seconds_total"]) > 0.0
    assert set(xo) == set(BENCH_SWEEP["sizes"])
    for size, n_star in xo.items():
        expect = None
        for n in sorted(BENCH_SWEEP["frame_counts"]):
            cells = [x for x in rows if int(x["width"]) == size and int(x["N"]) == n and x["seconds_total"] != "nan"]
            w = next((x for x in cells if x["algorithm"] == "with_ft"), None)
            wo = next((x for x in cells if x["algorithm"] == "without_ft"), None)
            if w and wo and float(w["seconds_total"]) < float(wo["seconds_total"]):
                expect = n
                break
        assert n_star == expect
    echo = json.loads((tmp_path / "run.json").read_text())
    assert echo["subcommand"] == "bench" and echo["budgets"] == "1073741824,40000,100"


def test_out_dir_runs_assemble_the_partials_they_write(ddm, tmp_path):
    """With a workspace and no before_merge hook the map is assembled from the values the
    partials are written from; it equals the in-memory run and the files re-merge to it
    (grouped, cutoff and whole-plane layouts)."""
    st = ddm.generate(48, 40, 64, particles=20, seed=5)
    for qm, budget in ((None, 1 << 40), (9.5, 1 << 40), (None, 64 * 16 * 300), (11.0, 64 * 16 * 50)):
        base = ddm.RunConfig(precision="f64", q_max=qm, memory_bytes=budget)
        ref_map = ddm.run(st, base).values
        out = tmp_path / f"w{qm}_{budget}"
        cfg = ddm.RunConfig(precision="f64", q_max=qm, memory_bytes=budget, out_dir=str(out))
        got = ddm.run(st, cfg).values
        assert np.array_equal(got, ref_map)
        groups = O.plan_with_ft(len(O.cutoff_set(48, 40, qm)), 64, budget)[1]
        assert len(list((out / "partials").iterdir())) == len(groups)
        assert len(groups) > 1 or budget == 1 << 40


def test_stale_partials_in_out_dir_fail_as_the_reference(ddm, tmp_path):
    """A foreign group file in out_dir/partials makes the merge fail (`archive.cpp:239-262`)."""
    st = ddm.generate(32, 32, 32, particles=20, seed=6)
    out = tmp_path / "o"
    (out / "partials").mkdir(parents=True)
    (out / "partials" / "group9.bin").write_bytes(b"not a partial\n")
    with pytest.raises(ddm.InputError):
        ddm.run(st, ddm.RunConfig(memory_bytes=1 << 40, out_dir=str(out)))


# ----------------------------------------------------------------- `ddm compare`

@pytest.mark.parametrize("prec, algs", [("f64", ("with_ft", "without_ft")), ("f32", ("with_ft", "without_ft")),
                                        ("f64", ("with_ft", "direct"))])
def test_compare_agrees_with_its_own_runs(ddm, tmp_path, prec, algs):
    """`ddm compare` (`ddm_cli.cpp:247-290`): the deviation is max|a-b| / max(|a|,|b|) of the
    two algorithms' maps (`:132-141`), within the CLI's tolerance; the reference's own pair of
    runs on the same stack deviates within the same tolerance."""
    path = ddm.synth(str(tmp_path / "s"), size=32, frames=48, particles=20, seed=3)
    cfg = ddm.RunConfig(precision=prec, memory_bytes=1 << 40)
    rep = ddm.compare(path, cfg, algorithms=algs, out=str(tmp_path / "o"))
    maps = [ddm.run_raw_stack(path, ddm.RunConfig(algorithm=a, precision=prec, memory_bytes=1 << 40)).values
            for a in algs]
    peak = max(np.abs(maps[0]).max(), np.abs(maps[1]).max())
    assert rep["deviation"] == pytest.approx(np.abs(maps[0] - maps[1]).max() / peak, rel=1e-12, abs=0)
    assert rep["tolerance"] == (1e-4 if prec == "f32" else 1e-9) and rep["pass"]
    saved = json.loads((tmp_path / "o" / "compare.json").read_text())
    assert saved["pass"] and saved["algorithms"] == list(algs) and saved["deviation"] == rep["deviation"]


def test_widened_f32_download_is_bit_identical(ddm, tmp_path):
    """DDM_D2H_WIDEN=1: the f32 device map widened on the host (exact) equals the f64 device
    map path bit for bit where the temporal engine computes d in f32 (the register engines,
    N = 1024 here; a map above the 4 M-value threshold)."""
    import subprocess
    import sys
    st = ddm.generate(128, 64, 1024, particles=40, seed=9)
    np.save(tmp_path / "st.npy", st)
    code = ("import numpy as np, sys; sys.path.insert(0, '.'); from paper_2012_05695_b200 import ddm; "
            f"st = np.load('{tmp_path}/st.npy'); a = ddm.run(st, ddm.RunConfig(precision='f32', memory_bytes=1 << 40)); "
            f"np.save('{tmp_path}/w.npy', a.values)")
    root = Path(__file__).resolve().parents[1]
    env = dict(__import__("os").environ, DDM_D2H_WIDEN="1")
    subprocess.run([sys.executable, "-c", code], cwd=root, env=env, check=True, timeout=300)
    ref = ddm.run(st, ddm.RunConfig(precision="f32", memory_bytes=1 << 40)).values
    assert ref.size >= 1 << 22
    assert np.array_equal(np.load(tmp_path / "w.npy"), ref)


def test_bench_counters_scale_as_the_reference_expects(ddm):
    """`test_bench.cpp:66-107`: WITHOUT_FT pairs N(N-1)/2, WITH_FT one group with two temporal
    transforms per wave vector (8 x 5 at 8^2) and N spatial transforms; counters never
    shrink as N grows."""
    rows, _ = ddm.bench_sweep((8, 16, 32, 256, 512), (8,), repetitions=1, warmup=0)
    cell = {(r["algorithm"], int(r["N"])): r for r in rows}
    assert int(cell[("without_ft", 256)]["count_pairs"]) == 256 * 255 // 2
    assert int(cell[("without_ft", 512)]["count_pairs"]) == 512 * 511 // 2
    f = cell[("with_ft", 256)]
    assert int(f["groups_or_passes"]) == 1 and int(f["count_temporal_ffts"]) == 2 * 8 * 5
    assert int(f["count_spatial_ffts"]) == 256
    for alg in ("with_ft", "without_ft"):
        sp = [int(cell[(alg, n)]["count_spatial_ffts"]) for n in (8, 16, 32, 256, 512)]
        pr = [int(cell[(alg, n)]["count_pairs"]) for n in (8, 16, 32, 256, 512)]
        assert sp == sorted(sp) and pr == sorted(pr)
        assert all(float(cell[(alg, n)]["seconds_total"]) > 0 for n in (8, 16, 32, 256, 512))

"""Readers for the `ddm analyze` artefact set (`proj/tools/ddm_cli.cpp:206-240`): the per-lag
maps d_m<lag>.bin (raw little-endian f64, H x (W/2+1)), index.json (`archive.cpp:60-110`),
radial.csv and fits.csv (`analysis.cpp:273-304`).  Test infrastructure."""
from __future__ import annotations

import csv
import json
from pathlib import Path

import numpy as np

VOLATILE_INDEX_KEYS = ("timing", "tool_version")


def read_artifacts(out_dir) -> dict:
    out = Path(out_dir)
    index = json.loads((out / "index.json").read_text())
    hc = int(index["half_cols"])
    maps = {int(m["lag"]): np.fromfile(out / m["file"], dtype="<f8").reshape(int(index["height"]), hc)
            for m in index["maps"]}
    with open(out / "radial.csv", newline="") as f:
        rows = list(csv.reader(f))
    assert rows[0] == ["lag", "q_bin", "mean", "count"]
    radial = [(int(r[0]), int(r[1]), float(r[2]), int(r[3])) for r in rows[1:]]
    fits = None
    if (out / "fits.csv").exists():
        with open(out / "fits.csv", newline="") as f:
            rows = list(csv.reader(f))
        assert rows[0] == ["q_bin", "A", "B", "tau_seconds", "residual", "flag"]
        fits = [(int(r[0]), float(r[1]), float(r[2]), float(r[3]), float(r[4]), r[5]) for r in rows[1:]]
    files = sorted(p.name for p in out.iterdir() if p.is_file())
    return {"index": index, "maps": maps, "radial": radial, "fits": fits, "files": files}


def stable_index(index: dict) -> dict:
    return {k: v for k, v in index.items() if k not in VOLATILE_INDEX_KEYS}

"""Wall time of `ddm analyze` (ddm_b200_analyze) on a synthetic raw stack, split into the
run (device + host map) and the artefact writing, against the reference library's own
analyze on a bounded sample when oracle/_ref is present.

    python tools/bench_analyze.py [W H N [precision [lag_spec]]]
"""
import json
import os
import shutil
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from golden.make_golden import write_stack  # noqa: E402
from oracle import ddm_oracle as O  # noqa: E402
from paper_2012_05695_b200 import ddm  # noqa: E402


def main():
    a = sys.argv[1:]
    w, h, n = (int(x) for x in a[:3]) if len(a) >= 3 else (512, 512, 1024)
    prec = a[3] if len(a) > 3 else "f32"
    lag_spec = a[4] if len(a) > 4 else "all"
    lags = O.log_lags(n) if lag_spec == "log" else []
    tmp = Path(tempfile.mkdtemp(dir=os.environ.get("TMPDIR", "/tmp")))
    st = ddm.generate(w, h, n, particles=100, diffusion=0.5, seed=7)
    src = tmp / "in.raw"
    write_stack(src, "raw_stack", st)
    cfg = ddm.RunConfig(precision=prec, lags=lags, memory_bytes=1 << 40, workers=8)
    res = {}
    for rep in range(3):
        out = tmp / f"out{rep}"
        t0 = time.perf_counter()
        info = ddm.analyze(str(src), str(out), cfg)
        wall = time.perf_counter() - t0
        size = sum(p.stat().st_size for p in out.iterdir() if p.is_file())
        res = {"W": w, "H": h, "N": n, "precision": prec, "lags": lag_spec, "wall_s": wall,
               "run_total_s": info["timing"]["total"], "write_s": wall - info["timing"]["total"],
               "artefact_bytes": size, "write_GBps": size / max(wall - info["timing"]["total"], 1e-9) / 1e9,
               "frames_per_s": n / wall}
        shutil.rmtree(out)
    print(json.dumps(res), flush=True)
    shutil.rmtree(tmp)


if __name__ == "__main__":
    main()

"""The paper's WITH_FT / WITHOUT_FT crossover (acceptance 5) on the device:
`ddm bench` over N x size through ddm_b200_bench_sweep (f64 cells, medians of 3 after one
warm-up), bench.csv + the crossover N* per size into OUT (default gpurun_out/crossover).

    python tools/crossover.py [OUT]
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2012_05695_b200 import ddm  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/crossover"
rows, xo = ddm.bench_sweep(frame_counts=(16, 32, 64, 128, 256, 512, 1024), sizes=(32, 64, 128, 256),
                           algorithms=("with_ft", "without_ft"), workers=(2,), repetitions=3, warmup=1,
                           out=out)
print(json.dumps({"crossover_n_star": xo}))
for r in rows:
    print(r["algorithm"], r["N"], r["width"], r["seconds_total"], r["seconds_step1"], r["seconds_step2"])

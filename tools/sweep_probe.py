"""Print the release gate's crossover sweep (criterion 5, `acceptance_main.cpp:221-270`) as
the device path times it: per cell the median TimingBreakdown phases (ms)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2012_05695_b200 import ddm  # noqa: E402

for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    rows, nstar = ddm.bench_sweep([256, 512, 1024, 2048, 4096], [64], repetitions=3, warmup=1)
    print(f"sweep {rep}: N* = {nstar}")
    for r in rows:
        print("  {:10s} N={:5s} total={:8.3f} disk={:7.3f} s1={:7.3f} s2={:7.3f} merge={:7.3f}".format(
            r["algorithm"], r["N"], *(1e3 * float(r[k]) for k in
                                            ("seconds_total", "seconds_disk", "seconds_step1",
                                             "seconds_step2", "seconds_merge"))))

"""Aggregate an ncu `--page source --csv` (SASS view) by opcode: executed warp instructions
and stall samples (long/short scoreboard, wait, mio...)."""
import csv
import collections
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    agg = collections.defaultdict(lambda: collections.Counter())
    tot = collections.Counter()
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        op = r[ix["Source"]].strip().split()
        if not op:
            continue
        o = op[0]
        if o.startswith("@"):
            o = op[1] if len(op) > 1 else o
        o = o.split(".")[0]
        def num(k):
            try:
                return float(r[ix[k]].replace(",", "")) if k in ix and r[ix[k]] else 0.0
            except ValueError:
                return 0.0
        c = agg[o]
        c["inst"] += num("Instructions Executed")
        c["samples"] += num("Warp Stall Sampling (All Samples)")
        for k in ("stall_long_sb", "stall_short_sb", "stall_wait", "stall_mio", "stall_selected",
                  "stall_not_selected", "stall_math", "stall_barrier", "stall_lg", "stall_dispatch",
                  "stall_no_inst", "stall_branch_resolving"):
            c[k] += num(k)
        for k, v in c.items():
            pass
    for c in agg.values():
        tot.update(c)
    print(f"total inst {tot['inst']:.4g}  samples {tot['samples']:.4g}")
    keys = ["inst", "samples", "stall_selected", "stall_long_sb", "stall_short_sb", "stall_wait",
            "stall_mio", "stall_not_selected", "stall_barrier", "stall_lg", "stall_no_inst"]
    print(f"{'op':10s}" + "".join(f"{(k[6:] if k.startswith('stall_') else k):>13s}" for k in keys))
    for o, c in sorted(agg.items(), key=lambda kv: -kv[1]["inst"])[:top]:
        print(f"{o:10s}" + "".join(f"{c[k]:13.4g}" for k in keys))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)

"""Summarise one GPU round (tools/gpu_round.sh outputs in gpurun_out/) into profiles/.

    python tools/profile_summary.py r01a [kernel ...]

Writes profiles/<tag>_summary.md (bench line, ncu launch list per kernel, per-kernel ncu
--set full key metrics, SASS opcode mix of the top kernel), copies the raw ncu CSVs and
updates profiles/ncu_traffic.json ({stage: dram bytes per launch}) which bench.py reports as
roofline.traffic.
"""
import collections
import csv
import io
import json
import shutil
import sys
from contextlib import redirect_stdout
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"
sys.path.insert(0, str(ROOT / "tools"))

STAGE = {"temporal": "temporal", "rows": "spatial", "cols": "spatial", "spatial": "spatial"}

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct"]


def launches(tag):
    p = OUT / f"launches_{tag}.csv"
    rows = [r for r in csv.reader(open(p)) if len(r) > 5]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]]
        short = name.split("(")[0].replace("void ", "")
        agg.setdefault(short, []).append(float(r[ix["Metric Value"]].replace(",", "")) / 1e3)
    return agg


def raw(tag, k):
    p = OUT / f"raw_{k}_{tag}.csv"
    if not p.exists():
        return None
    rows = list(csv.reader(open(p)))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


def main(tag, kernels):
    PROF.mkdir(exist_ok=True)
    md = [f"# GPU round `{tag}` (B200, one GPU)\n"]
    for name in (f"gpu_{tag}.txt",):
        if (OUT / name).exists():
            md += ["```", (OUT / name).read_text().strip(), "```\n"]
    b = OUT / f"bench_{tag}.json"
    if b.exists():
        md += ["## bench.py line\n", "```json", b.read_text().strip(), "```\n"]
    rb = OUT / f"bench_ref_{tag}.json"
    if rb.exists():
        md += ["## bench.py --impl reference\n", "```json", rb.read_text().strip().splitlines()[-1], "```\n"]
    if (OUT / f"launches_{tag}.csv").exists():
        agg = launches(tag)
        md += ["## ncu launch list (`--metrics gpu__time_duration.sum --clock-control none`, "
               "`bench.py --steps 2 --warmup 1`; cold, serialised)\n",
               "| kernel | launches | mean us | total us | share |", "|---|---|---|---|---|"]
        tot = sum(sum(v) for v in agg.values())
        for k, v in agg.items():
            md.append(f"| `{k}` | {len(v)} | {sum(v)/len(v):.2f} | {sum(v):.1f} | {sum(v)/tot:.1%} |")
        md.append("")
        shutil.copy(OUT / f"launches_{tag}.csv", PROF / f"{tag}_launches.csv")
    traffic_p = PROF / "ncu_traffic.json"
    traffic = json.loads(traffic_p.read_text()) if traffic_p.exists() else {}
    for k in kernels:
        r = raw(tag, k)
        if not r:
            continue
        d, u = r
        md += [f"## `{k}` — ncu --set full (one launch)\n", "| metric | value | unit |", "|---|---|---|"]
        for key in KEYS:
            if key in d:
                md.append(f"| {key} | {d[key]} | {u.get(key, '')} |")
        md.append("")
        shutil.copy(OUT / f"raw_{k}_{tag}.csv", PROF / f"{tag}_raw_{k}.csv")
        try:
            rd = float(d["dram__bytes_read.sum"].replace(",", "")) * (1e9 if "G" in u["dram__bytes_read.sum"] else 1e6 if "M" in u["dram__bytes_read.sum"] else 1e3 if "K" in u["dram__bytes_read.sum"] else 1)
            wr = float(d["dram__bytes_write.sum"].replace(",", "")) * (1e9 if "G" in u["dram__bytes_write.sum"] else 1e6 if "M" in u["dram__bytes_write.sum"] else 1e3 if "K" in u["dram__bytes_write.sum"] else 1)
            stage = next(v for s, v in STAGE.items() if s in k)
            rec = {"dram_bytes": rd + wr, "stage": stage}
            if "smsp__inst_executed.sum" in d:
                rec["warp_inst"] = float(d["smsp__inst_executed.sum"].replace(",", ""))
            traffic.setdefault(tag, {})[k] = rec
        except Exception:
            pass
        src = OUT / f"source_{k}_{tag}.csv"
        if src.exists():
            import sass_profile
            buf = io.StringIO()
            with redirect_stdout(buf):
                sass_profile.main(str(src), 25)
            md += [f"SASS opcode mix (warp instructions executed, stall samples) of `{k}`:\n",
                   "```", buf.getvalue().rstrip(), "```\n"]
    traffic["latest"] = tag
    traffic_p.write_text(json.dumps(traffic, indent=1))
    (PROF / f"{tag}_summary.md").write_text("\n".join(md) + "\n")
    print(PROF / f"{tag}_summary.md")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:] or ["temporal_warp_kernel", "rows2_kernel", "cols2_kernel"])

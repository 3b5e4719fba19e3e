"""Summarise an ncu raw CSV (one kernel): key throughput / stall metrics."""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "l1tex__t_bytes.sum"]
STALL = "smsp__average_warp_latency_issue_stalled_"


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    for k in KEYS:
        if k in d:
            print(f"{k:70s} {d[k]} {u.get(k, '')}")
    stalls = sorted(((float(d[k].replace(',', '')), k[len(STALL):]) for k in hdr
                     if k.startswith(STALL) and k.endswith("ratio") and d[k] not in ("", "n/a")),
                    reverse=True)[:10]
    print("top stalls (ratio):", ", ".join(f"{n}={v:.2f}" for v, n in stalls))
    other = sorted(((k, d[k]) for k in hdr if "warp_latency_issue_stalled" in k), key=lambda x: x[0])
    if not stalls:
        for k, v in other[:40]:
            print(k, v)


if __name__ == "__main__":
    main(sys.argv[1])

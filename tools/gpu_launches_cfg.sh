mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${1:-c3}.csv python bench.py --config ${1:-c3} --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/c3l.log 2>&1
echo rc=$?
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/launches_${1:-c3}.csv")))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            k = d["Kernel Name"][:90]
            v = float(d["Metric Value"].replace(",", ""))
            u = d.get("Metric Unit", "")
            v = v / 1e3 if u == "usecond" else (v / 1e6 if u == "nsecond" else v)
            agg[k][0] += 1; agg[k][1] += v
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:12]:
    print(f"{t:9.3f} ms {n:4d}x {k}")
PY

"""Per-block breakdown of an ncu SASS source CSV: samples and executed warp-instructions."""
import collections
import csv
import sys

path, W = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 150
norm = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
rows = list(csv.reader(open(path)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) > 5]
ci = {h: i for i, h in enumerate(hdr)}
S, E = ci['Warp Stall Sampling (All Samples)'], ci['Instructions Executed']
tot = sum(int(r[S] or 0) for r in data)
tex = sum(int(r[E] or 0) for r in data)
print('samples', tot, 'warp-instr', tex, 'per unit', tex / norm)


def op(r):
    t = r[1].split()
    o = t[1] if t and t[0].startswith('@') and len(t) > 1 else (t[0] if t else '')
    return o.split('.')[0]


for i in range(0, len(data), W):
    blk = data[i:i + W]
    s = sum(int(r[S] or 0) for r in blk)
    ex = sum(int(r[E] or 0) for r in blk)
    if s == 0 and ex == 0:
        continue
    ops = collections.Counter(op(r) for r in blk)
    print(f"{i:5d} samp {100*s/tot:5.1f}%  exec/unit {ex/norm:9.1f}  {dict(ops.most_common(6))}")

# stall reasons per block (second table)
reasons = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
print('\nblock  ' + ' '.join(f"{r[6:12]:>7s}" for r in reasons))
for i in range(0, len(data), W):
    blk = data[i:i + W]
    vals = [sum(int(r[ci[x]] or 0) for r in blk) for x in reasons]
    if sum(vals) == 0:
        continue
    print(f"{i:5d}  " + ' '.join(f"{100*v/tot:7.1f}" for v in vals))

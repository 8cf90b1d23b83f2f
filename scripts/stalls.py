"""Aggregate ncu source-page stall samples by code region (index ranges) and reason.
usage: python scripts/stalls.py src.csv [lo hi ...]"""
import csv
import sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
seen, data = set(), []
for r in rows[2:]:
    if r and r[0].startswith('0x') and r[0] not in seen:
        seen.add(r[0]); data.append(r)
reasons = [h for h in hdr if h.startswith('stall_') and '(Not' not in h]
ri = {h: hdr.index(h) for h in reasons}
i_src = hdr.index("Source")
tot = sum(int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0) for r in data)
def agg(lo, hi):
    s = {h: sum(int(r[ri[h]] or 0) for r in data[lo:hi]) for h in reasons}
    t = sum(s.values())
    return t, sorted(((v, h) for h, v in s.items() if v), reverse=True)[:6]
print("total", tot, "instructions", len(data))
b = [int(x) for x in sys.argv[2:]] or [0, len(data)]
for lo, hi in zip(b[::2], b[1::2]):
    t, top = agg(lo, hi)
    print(f"[{lo},{hi}) {t} ({100*t/max(tot,1):.1f}%)", [(h, v) for v, h in top])
if len(sys.argv) > 2 and sys.argv[-1] == 'list':
    pass

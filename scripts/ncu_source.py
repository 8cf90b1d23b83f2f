"""Summarise an ncu source page (SASS view): per-instruction shared-memory excess wavefronts and
warp-stall samples, aggregated by opcode and listing the hottest instructions.

    ncu -i rep --page source --csv --kernel-name regex:K --print-source sass > src.csv
    python scripts/ncu_source.py src.csv [top]
"""
import csv
import sys
from collections import defaultdict


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    idx = {n: i for i, n in enumerate(h)}
    data = [r for r in rows[2:] if len(r) == len(h) and r[idx["Address"]] != "Address"]

    def num(r, k):
        if k not in idx:
            return 0.0
        try:
            return float(r[idx[k]].replace(",", "") or 0)
        except ValueError:
            return 0.0
    stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    tot = sum(num(r, "Warp Stall Sampling (All Samples)") for r in data)
    print(f"instructions {len(data)}, stall samples {tot:.0f}")
    by_op = defaultdict(lambda: defaultdict(float))
    for r in data:
        op = r[idx["Source"]].split()[0] if r[idx["Source"]].split() else "?"
        if op.startswith("@"):
            op = r[idx["Source"]].split()[1]
        op = op.split(".")[0]
        by_op[op]["samples"] += num(r, "Warp Stall Sampling (All Samples)")
        by_op[op]["excess_wavefronts"] += num(r, "L1 Wavefronts Shared Excessive")
        by_op[op]["executed"] += num(r, "Instructions Executed")
        for c in stall_cols:
            by_op[op][c] += num(r, c)
    print("\nby opcode (stall samples share, top stall reasons, excess smem wavefronts):")
    for op, d in sorted(by_op.items(), key=lambda kv: -kv[1]["samples"])[:top]:
        reasons = sorted(((d[c], c[6:]) for c in stall_cols), reverse=True)[:3]
        print(f"  {op:10s} {100 * d['samples'] / max(tot, 1):5.1f}%  exec {d['executed']:.3g}  "
              f"excess_wf {d['excess_wavefronts']:.3g}  " + ", ".join(f"{n} {100 * v / max(tot, 1):.1f}%" for v, n in reasons))
    print("\nhottest instructions:")
    for r in sorted(data, key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))[:top]:
        reasons = sorted(((num(r, c), c[6:]) for c in stall_cols), reverse=True)[:2]
        print(f"  {r[idx['Address']]:>8s} {100 * num(r, 'Warp Stall Sampling (All Samples)') / max(tot, 1):5.2f}%  "
              f"{r[idx['Source']][:60]:60s} " + ", ".join(f"{n} {v:.0f}" for v, n in reasons))
    conf = [r for r in data if num(r, "L1 Wavefronts Shared Excessive") > 0]
    if conf:
        print("\ninstructions with excess shared wavefronts:")
        for r in sorted(conf, key=lambda r: -num(r, "L1 Wavefronts Shared Excessive"))[:top]:
            print(f"  {r[idx['Address']]:>8s} excess {num(r, 'L1 Wavefronts Shared Excessive'):.3g} "
                  f"wf {num(r, 'L1 Wavefronts Shared'):.3g} ideal {num(r, 'L1 Wavefronts Shared Ideal'):.3g}  "
                  f"{r[idx['Source']][:70]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)

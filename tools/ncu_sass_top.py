"""Summarise an `ncu --page source --csv --print-source sass` export: stall
samples and executed instructions per opcode, and the top stalled lines.

    python tools/ncu_sass_top.py export.csv [n_top]
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    n_top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    rows = list(csv.reader(open(path)))
    h = rows[1]
    data = rows[2:]
    ia, isrc = h.index("Address"), h.index("Source")
    iss = h.index("Warp Stall Sampling (All Samples)")
    iex = h.index("Instructions Executed")
    ex, smp = collections.Counter(), collections.Counter()
    for r in data:
        op = r[isrc].split()
        if not op:
            continue
        o = (op[1] if op[0].startswith("@") else op[0]).split(".")[0]
        ex[o] += float(r[iex] or 0)
        smp[o] += float(r[iss] or 0)
    T, S = sum(ex.values()), sum(smp.values())
    print(f"warp instructions {T:.3e}, stall samples {S:.0f}")
    for o, v in ex.most_common(25):
        print(f"  {o:10s} {v / 1e6:8.2f}M {100 * v / T:5.1f}%  samples {100 * smp[o] / S:5.1f}%")
    print("top stalled instructions:")
    for r in sorted(data, key=lambda r: -float(r[iss] or 0))[:n_top]:
        print(f"  {r[ia][-5:]} {100 * float(r[iss]) / S:5.1f}% ex={r[iex]:>9} {r[isrc][:80]}")


if __name__ == "__main__":
    main()

"""Attribute ncu SASS-level stall samples / executed instructions to CUDA
source lines, using `nvdisasm -g` line info of the same cubin.

    python tools/ncu_lines.py export_sass.csv kernel.cubin mangled_name [n_top]
"""
import collections
import csv
import re
import subprocess
import sys


def line_map(cubin, fn):
    out = subprocess.run(["nvdisasm", "-g", "-c", "-fun", fn, cubin], capture_output=True,
                         text=True).stdout
    if not out.strip():
        out = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
        a = out.find(".text." + fn)
        out = out[a:]
        b = out.find("//---------------------", 10)
        out = out[:b] if b > 0 else out
    m, line = {}, None
    for ln in out.splitlines():
        g = re.search(r"//## File \".*?\", line (\d+)", ln)
        if g:
            line = int(g.group(1))
            continue
        g = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if g and line is not None:
            m[int(g.group(1), 16)] = line
    return m


def main():
    path, cubin, fn = sys.argv[1:4]
    n_top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    rows = list(csv.reader(open(path)))
    h, data = rows[1], rows[2:]
    ia, iss, iex = (h.index("Address"), h.index("Warp Stall Sampling (All Samples)"),
                    h.index("Instructions Executed"))
    base = min(int(r[ia], 16) for r in data)
    lm = line_map(cubin, fn)
    reasons = [(i, c[6:]) for i, c in enumerate(h) if c.startswith("stall_") and "(" not in c]
    smp, ex = collections.Counter(), collections.Counter()
    why = collections.defaultdict(collections.Counter)
    tot_why = collections.Counter()
    for r in data:
        off = int(r[ia], 16) - base
        ln = lm.get(off, -1)
        smp[ln] += float(r[iss] or 0)
        ex[ln] += float(r[iex] or 0)
        for i, name in reasons:
            v = float(r[i] or 0)
            why[ln][name] += v
            tot_why[name] += v
    S, T = sum(smp.values()), sum(ex.values())
    print(f"samples {S:.0f}, warp instructions {T:.3e}")
    print("stall reasons:", ", ".join(f"{k} {100 * v / S:.1f}%" for k, v in tot_why.most_common(8)))
    for ln, v in smp.most_common(n_top):
        top = ", ".join(f"{k} {100 * x / max(v, 1):.0f}%" for k, x in why[ln].most_common(3))
        print(f"  line {ln:5d}: {100 * v / S:5.1f}% samples, {100 * ex[ln] / T:5.1f}% instr  [{top}]")


if __name__ == "__main__":
    main()

"""Attribute ncu SASS stall samples to the kernel's own source lines, folding
inlined helpers (tcgen05.cuh waits, exp2, ...) into their CALL SITE.

    python tools/ncu_callsite.py export_sass.csv all.sass kernel_mangled_name [n_top]

export_sass.csv: `ncu -i rep --page source --csv --print-source sass` of ONE
kernel; all.sass: `nvdisasm -g -gi -c <cubin>` of the same build.
"""
import collections
import csv
import re
import sys


def call_sites(sass_path, fn, main_file="attn_tc.cu"):
    lines = open(sass_path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith("//---") and f".text.{fn} " in l)
    m, cur = {}, None
    for l in lines[start + 1:]:
        if l.startswith("//---------------------"):
            break
        g = re.search(r'//## File "(.*?)", line (\d+)(?: inlined at "(.*?)", line (\d+))?', l)
        if g:
            f, ln, fi, li = g.groups()
            if fi and fi.endswith(main_file):
                cur = int(li)
            elif f.endswith(main_file):
                cur = int(ln)
            continue
        g = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
        if g and cur is not None:
            m[int(g.group(1), 16)] = cur
    return m


def main():
    exp, sass, fn = sys.argv[1:4]
    n_top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    rows = list(csv.reader(open(exp)))
    h = rows[1]
    data = rows[2:]
    ia, iss, iex = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), \
        h.index("Instructions Executed")
    base = min(int(r[ia], 16) for r in data)
    cs = call_sites(sass, fn)
    smp, ex = collections.Counter(), collections.Counter()
    for r in data:
        off = int(r[ia], 16) - base
        ln = cs.get(off, -1)
        smp[ln] += float(r[iss] or 0)
        ex[ln] += float(r[iex] or 0)
    S, T = sum(smp.values()), sum(ex.values())
    src = {}
    for ln, v in smp.most_common(n_top):
        print(f"  attn line {ln:5d}: {100 * v / S:5.1f}% samples  {100 * ex[ln] / T:5.1f}% instr")


if __name__ == "__main__":
    main()

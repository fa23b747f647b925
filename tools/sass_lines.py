"""Executed warp instructions per source line: joins an ncu SASS page
(`ncu -i rep --page source --csv --print-source sass`) with `nvdisasm -g -c`
line info of the same cubin.
    python tools/sass_lines.py sass.csv disasm.txt <mangled-substring> [per-unit-divisor] [top]"""
import collections
import csv
import re
import sys


def main():
    sass_csv, dis, fn = sys.argv[1], sys.argv[2], sys.argv[3]
    div = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
    lines = open(dis).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith(".text.") and fn in l and l.endswith(":"))
    cur = "?"
    off2line = {}
    for l in lines[start + 1:]:
        if l.startswith(".text.") or l.startswith("//-----"):
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = m.group(1).split("/")[-1] + ":" + m.group(2)
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m:
            off2line[int(m.group(1), 16)] = (cur, m.group(2))
    rows = list(csv.reader(open(sass_csv)))
    hdr = rows[1]
    i_a, i_e = hdr.index("Address"), hdr.index("Instructions Executed")
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    base = int(rows[2][i_a], 16)
    agg, st, ops = collections.Counter(), collections.Counter(), collections.defaultdict(collections.Counter)
    for r in rows[2:]:
        if len(r) <= i_e:
            continue
        off = int(r[i_a], 16) - base
        ln, ins = off2line.get(off, ("?", "?"))
        n = int(r[i_e] or 0)
        agg[ln] += n
        st[ln] += int(r[i_s] or 0)
        op = ins.split()[0] if ins else "?"
        if op.startswith("@"):
            op = ins.split()[1]
        ops[ln][op.split(".")[0]] += n
    tot, stot = sum(agg.values()), sum(st.values()) or 1
    for ln, n in agg.most_common(top):
        mix = " ".join(f"{o}:{c / div:.0f}" for o, c in ops[ln].most_common(4))
        print(f"{n / div:9.1f} {100 * n / tot:5.1f}% stall {100 * st[ln] / stot:5.1f}%  {ln:22s} {mix}")
    print("total per unit", tot / div)


if __name__ == "__main__":
    main()

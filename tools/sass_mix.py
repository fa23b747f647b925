"""Executed-instruction mix per opcode from `ncu --page source --csv --print-source sass`.
    python tools/sass_mix.py sass.csv [top]"""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr = rows[1]
    i_src, i_ex = hdr.index("Source"), hdr.index("Instructions Executed")
    i_st = hdr.index("Warp Stall Sampling (All Samples)")
    agg = collections.Counter()
    stall = collections.Counter()
    tot = 0
    for r in rows[2:]:
        if len(r) <= i_ex:
            continue
        src = r[i_src].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        n = int(r[i_ex] or 0)
        agg[op] += n
        stall[op] += int(r[i_st] or 0)
        tot += n
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    st = sum(stall.values()) or 1
    for op, n in agg.most_common(top):
        print(f"{op:12s} {n:14d} {100 * n / tot:5.1f}%  stall-samples {100 * stall[op] / st:5.1f}%")
    print("total", tot)


if __name__ == "__main__":
    main()

"""Per-CUDA-source-line totals from an ncu report (needs -lineinfo and
--import-source on):  python tools/ncu_lines.py <rep> [top] [kernel-substring]"""

import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    filt = sys.argv[3] if len(sys.argv) > 3 else ""
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    path, func, hdr = "", "", None
    agg = []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            func = r[1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0] or (filt and filt not in func):
            continue
        try:
            ie = float(r[hdr.index("Instructions Executed")] or 0)
            ws = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except (ValueError, IndexError):
            continue
        agg.append((ie, ws, f"{path}:{r[0]}", r[1].strip()[:80]))
    ti = sum(a[0] for a in agg) or 1
    ts = sum(a[1] for a in agg) or 1
    print(f"total warp-instructions {ti:.3g}, stall samples {ts:.0f}")
    print("-- by instructions")
    for ie, ws, loc, src in sorted(agg, reverse=True)[:top]:
        print(f"{100 * ie / ti:5.1f}% inst {100 * ws / ts:5.1f}% stall  {loc:22s} {src}")
    print("-- by stall samples")
    for ie, ws, loc, src in sorted(agg, key=lambda a: -a[1])[:top // 2]:
        print(f"{100 * ie / ti:5.1f}% inst {100 * ws / ts:5.1f}% stall  {loc:22s} {src}")


if __name__ == "__main__":
    main()

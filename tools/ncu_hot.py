"""Summarise an ncu report: per kernel, the SASS instructions with the most
warp-stall samples (needs a capture with --set full --import-source on).

    python tools/ncu_hot.py gpurun_out/net.ncu-rep [top] [kernel-substring]
"""

import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    filt = sys.argv[3] if len(sys.argv) > 3 else ""
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks, cur = [], None
    for line in txt.splitlines():
        if line.startswith('"Kernel Name"'):
            cur = [line.split('","')[1].rstrip('",'), []]
            blocks.append(cur)
        elif cur is not None:
            cur[1].append(line)
    for name, lines in blocks:
        if filt and filt not in name:
            continue
        rows = list(csv.reader(io.StringIO("\n".join(lines))))
        hdr, data = rows[0], rows[1:]
        i_src, i_s = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
        stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h and i != i_s]
        total = sum(float(r[i_s] or 0) for r in data if len(r) > i_s)
        print(f"== {name[:110]}  samples={total:.0f}")
        data.sort(key=lambda r: -float(r[i_s] or 0) if len(r) > i_s else 0)
        for r in data[:top]:
            s = float(r[i_s] or 0)
            print(f"  {100 * s / max(total, 1):5.1f}%  {r[0][-5:]}  {r[i_src].strip()[:70]}")


if __name__ == "__main__":
    main()

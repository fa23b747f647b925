"""Write the committed profile summaries (profiles/<round>/) from raw ncu output.

    python tools/profile_summary.py <round> [--launches gpurun_out/launches.csv]
                                    [--rep gpurun_out/net.ncu-rep ...]

* launches.md : the `--metrics gpu__time_duration.sum` launch list of one
  bench.py run, aggregated per kernel (count, total, share of GPU time);
* <rep>.md    : per-kernel key metrics of a `--set full` capture (duration,
  DRAM bytes, DRAM throughput, issue/ALU utilisation, occupancy, smem bank
  conflicts, top stall reasons);
* traffic.json: DRAM bytes (read + write) per launch per kernel, read by
  bench.py for the roofline "traffic" field.
"""

from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import re
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%_of_peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_%"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_bank_conflicts"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_%"),
]


def short_name(name: str) -> str:
    I = r"(?:\(int\))?"
    m = re.search(rf"NetCfg<{I}(\d+), {I}(\d+), ([a-z ]+?), (?:nsg::)?([A-Za-z ]+?), {I}(\d), {I}(\d)(?:, {I}(\d+))?>",
                  name)
    if m:
        n, dag, u, p, mode, lay, g = m.groups()
        if g and g != "1":
            n = f"{int(n) * int(g)} ({g} lanes x {n})"
        fam = {"0": "best", "1": "bn", "2": "merge"}[dag]
        kt = "u64" if "long" in u else "u32"
        pt = {"NoPay": "keys", "unsigned int": "p32", "unsigned long": "p64"}.get(p.strip(), p)
        kind = "net_direct" if "net_direct_kernel" in name else "net_sort"
        return f"{kind} n={n} {fam} {kt} {pt} {'AoS' if lay == '1' else 'SoA'} {'UNIQUE' if mode == '1' else 'REF'}"
    pay_name = lambda p: {"NoPay": "keys", "unsigned int": "p32", "unsigned long": "p64"}.get(  # noqa: E731
        re.sub(r"^(?:nsg::)?", "", p.strip()), p.strip())
    m = re.search(rf"netbulk_kernel<{I}(\d+), {I}(\d), unsigned long, ((?:nsg::)?[A-Za-z ]+?), {I}(\d)", name)
    if m:
        n, dag, p, mode = m.groups()
        return f"netbulk n={n} {'best' if dag == '0' else 'bn'} u64 {pay_name(p)} SoA {'UNIQUE' if mode == '1' else 'REF'}"
    m = re.search(rf"nettma_kernel<{I}(\d), ((?:nsg::)?[A-Za-z ]+?), {I}(\d)>", name)
    if m:
        dag, p, mode = m.groups()
        return f"nettma n=16 {'best' if dag == '0' else 'bn'} u64 {pay_name(p)} SoA {'UNIQUE' if mode == '1' else 'REF'}"
    m = re.search(r"pksort_kernel<unsigned (long|int), ((?:nsg::)?[A-Za-z ]+?), (?:\(int\))?(\d), (?:\(int\))?(\d+), "
                  r"(?:\(bool\))?(\d|true|false), (?:nsg::)?(?:<unnamed>::)?(?:unnamed>::)?Phase(Bitonic|Rss)", name)
    if m:
        u, p, lg, e, full, ph = m.groups()
        return f"pksort {'merge' if ph == 'Bitonic' else 'rss'} NR={1 << int(lg)} {'u64' if u == 'long' else 'u32'} {pay_name(p)}"
    m = re.search(r"seg_kernel<unsigned (long|int), ((?:nsg::)?[A-Za-z ]+?), (?:\(int\))?(\d), (?:\(int\))?(\d), "
                  r"(?:\(int\))?(\d)>", name)
    if m:
        u, p, mode, dag, xk = m.groups()
        return (f"seg_kernel {'u64' if u == 'long' else 'u32'} {pay_name(p)} {'UNIQUE' if mode == '1' else 'REF'} "
                f"{'best' if dag == '0' else 'bn'} xform={['none', 'generic', 'float-desc'][int(xk)]}")
    return name[:90]


def launches(path: Path, out: Path):
    rows = list(csv.reader(io.StringIO("\n".join(l for l in path.read_text().splitlines()
                                                   if l.startswith('"')))))
    hdr = rows[0]
    i_name, i_val = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if len(r) <= i_val:
            continue
        v = float(r[i_val].replace(",", ""))
        unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "ns"
        ns = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "msecond": 1e6, "ms": 1e6, "nsecond": 1}.get(unit, 1)
        k = short_name(r[i_name])
        agg[k][0] += 1
        agg[k][1] += ns
    tot = sum(t for _, t in agg.values())
    lines = ["| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {k} | {c} | {t / 1e6:.3f} | {100 * t / tot:.1f} % |")
    out.write_text("# Launch list (ncu --metrics gpu__time_duration.sum --clock-control none)\n\n"
                   "Cold-cache, serialised per-launch times: compare SHARES, not absolutes.\n\n"
                   + "\n".join(lines) + "\n")


def rep_summary(rep: Path, out: Path, traffic: dict):
    """`rep`: an .ncu-rep, or the `--page raw --csv` export of one (*.raw.csv:
    reports with source are too large to bring back from the GPU box; a
    <stem>.lines.txt from tools/ncu_lines.py beside it is appended)."""
    if rep.suffix == ".csv":
        txt = rep.read_text()
    else:
        txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    lines = [f"# {rep.name} (ncu --set full --clock-control none)\n"]
    for r in rows[2:]:
        name = short_name(r[hdr.index("Kernel Name")])
        lines.append(f"## {name}\n")
        vals = {}
        for key, label in KEYS:
            if key in hdr:
                i = hdr.index(key)
                vals[label] = (r[i], units[i])
                lines.append(f"- {label}: {r[i]} {units[i]}")
        stalls = []
        for i, h in enumerate(hdr):
            if "smsp__pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued"):
                try:
                    stalls.append((float(r[i].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1
        lines.append("- top stalls: " + ", ".join(f"{h} {100 * v / tot:.0f}%"
                                                  for v, h in sorted(stalls, reverse=True)[:5]))
        lines.append("")
        try:
            def gb(label):
                v, u = vals[label]
                return float(v.replace(",", "")) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}.get(u, 1)
            traffic[name] = int(gb("dram_read") + gb("dram_write"))
        except Exception:
            pass
    lt = rep.with_name(rep.name.replace(".raw.csv", ".lines.txt"))
    if rep.suffix == ".csv" and lt.exists():
        head = lt.read_text().splitlines()[:28]
        lines += ["## CUDA source lines by warp instructions (tools/ncu_lines.py)\n", "```"] + head + ["```", ""]
    out.write_text("\n".join(lines) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("round")
    ap.add_argument("--launches", default=None)
    ap.add_argument("--rep", nargs="*", default=[])
    a = ap.parse_args()
    d = ROOT / "profiles" / a.round
    d.mkdir(parents=True, exist_ok=True)
    if a.launches:
        launches(Path(a.launches), d / "launches.md")
    tpath = ROOT / "profiles" / "traffic.json"
    traffic = json.loads(tpath.read_text()) if tpath.exists() else {}
    for rep in a.rep:
        rep_summary(Path(rep), d / (Path(rep).name.replace(".raw.csv", "").replace(".ncu-rep", "") + ".md"), traffic)
    tpath.write_text(json.dumps(traffic, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()

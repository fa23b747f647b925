"""Print the metrics that matter for a row-sorter kernel from an ncu report.
    python tools/ncu_peek.py gpurun_out/x.ncu-rep [extra-regex]"""
import csv
import io
import re
import subprocess
import sys

PAT = (r"gpu__time_duration.sum$|dram__bytes_(read|write).sum$|gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"
       r"|smsp__issue_active.avg.pct|sm__warps_active.avg.pct|launch__registers|launch__occupancy_limit"
       r"|l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum$|l1tex__data_pipe_lsu_wavefronts_mem_shared.sum$"
       r"|smsp__inst_executed.sum$|sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"
       r"|sm__inst_executed_pipe_lsu.avg.pct|launch__shared_mem_per_block_dynamic|launch__grid_size"
       r"|smsp__average_warp_latency_issue_stalled|l1tex__throughput.avg.pct|sm__pipe_shared_cycles_active.avg.pct"
       r"|smsp__inst_executed_op_shared|lts__t_sectors_srcunit_tex_op_(read|write).sum$")


def main():
    rep = sys.argv[1]
    extra = sys.argv[2] if len(sys.argv) > 2 else None
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print("==", r[hdr.index("Kernel Name")][:150])
        stalls = []
        for i, h in enumerate(hdr):
            if re.search(PAT, h) or (extra and re.search(extra, h)):
                print(f"  {h} = {r[i]} {units[i]}")
            if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
                try:
                    stalls.append((float(r[i].replace(",", "")), h[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1
        print("  stalls:", ", ".join(f"{h} {100 * v / tot:.0f}%" for v, h in sorted(stalls, reverse=True)[:8]))


if __name__ == "__main__":
    main()

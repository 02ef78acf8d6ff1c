"""Summarise ncu --set full reports: key metrics per launch and the top SASS
stall sites (needs -lineinfo). usage: python tools/ncu_summary.py rep.ncu-rep [...]"""
import csv
import io
import subprocess
import sys

KEYS = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
        "launch__occupancy_limit_registers", "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def raw(rep):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = (r[i], units[i])
        out.append(d)
    return out


def stalls(rep, top=25):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    heads = [i for i, r in enumerate(rows) if len(r) > 2 and r[0] == "Address"]
    if not heads:
        return []
    h = heads[-1]
    hdr = rows[h]
    S = hdr.index("Warp Stall Sampling (All Samples)")
    E = hdr.index("Instructions Executed")
    body = [r for r in rows[h + 1:] if len(r) == len(hdr) and r[0].startswith("0x")]
    tot = sum(int(r[S] or 0) for r in body) or 1
    top_rows = sorted(range(len(body)), key=lambda i: -int(body[i][S] or 0))[:top]
    return [(i, 100.0 * int(body[i][S]) / tot, body[i][E], body[i][1].strip()) for i in sorted(top_rows)]


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print("==", rep)
        for d in raw(rep):
            print("  " + " | ".join(f"{k.split('.')[0]}={v[0]}{'' if v[1] in ('', 'none') else ' ' + v[1]}"
                                    for k, v in d.items()))
        for i, pct, ex, ins in stalls(rep):
            print(f"   [{i:5d}] {pct:5.1f}%  x{ex:>9}  {ins[:90]}")

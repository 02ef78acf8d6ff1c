"""Stall samples of an ncu --set full capture aggregated by CUDA source line
(needs -lineinfo). usage: python tools/ncu_lines.py rep.ncu-rep [launch-skip] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
skip = sys.argv[2] if len(sys.argv) > 2 else "0"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--launch-skip",
                      skip, "--launch-count", "1"], capture_output=True, text=True).stdout
cur, hdr, res = None, None, {}
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        cur, hdr = r[1].split("/")[-1], None
        continue
    if r and r[0] in ("Line No", "#"):
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        try:
            s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        if s:
            res[(cur, d.get("Line No") or d.get("#"))] = s
tot = sum(res.values()) or 1
for (f, ln), s in sorted(res.items(), key=lambda x: -x[1])[:top]:
    print(f"{100 * s / tot:5.1f}%  {f}:{ln}")

"""Per-CUDA-source-line totals of one kernel in an ncu report (development
aid): stall samples and executed warp-instructions per line, from
  ncu -i rep --page source --csv --print-source cuda,sass
usage: python tools/ncu_src_lines.py rep.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, hdr, tot = None, None, {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("", "Function Name"):
        continue
    try:
        s = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        e = int(r[hdr.index("Instructions Executed")] or 0)
    except (ValueError, IndexError):
        continue
    key = (cur, int(r[0]))
    a = tot.setdefault(key, [0, 0, r[1].strip()[:90]])
    a[0] += s
    a[1] += e
S = sum(v[0] for v in tot.values()) or 1
E = sum(v[1] for v in tot.values()) or 1
print(f"samples {S}  warp-instructions {E:.4g}")
for (f, ln), (s, e, src) in sorted(tot.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * s / S:5.1f}% smp {100 * e / E:5.1f}% ins  {f}:{ln:<5} {src}")

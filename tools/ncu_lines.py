"""Per-SASS-instruction breakdown of one kernel in an ncu report: opcode
mix (executed warp-instructions) and the hottest instructions by stall
samples (in address order around them)."""
import csv, io, re, subprocess, sys
from collections import Counter
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
hdr = rows[hi]
ie, sm, src = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
th = hdr.index("Avg. Threads Executed")
data = []
for r in rows[hi + 1:]:
    try:
        data.append((int(r[ie] or 0), int(r[sm] or 0), float(r[th] or 0), r[src].strip()))
    except (ValueError, IndexError):
        pass
ti = sum(d[0] for d in data) or 1
ts = sum(d[1] for d in data) or 1
ops = Counter()
for n, _, _, s in data:
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", s)
    if m:
        ops[m.group(2)] += n
print(f"total warp-inst {ti:.3e}, stall samples {ts}")
print("opcode mix:", ", ".join(f"{k} {100*v/ti:.1f}%" for k, v in ops.most_common(22)))
hot = sorted(range(len(data)), key=lambda i: -data[i][1])[:top]
for i in sorted(hot):
    n, s_, t, s = data[i]
    print(f"{i:5d} inst {100*n/ti:5.2f}% stall {100*s_/ts:5.2f}% thr {t:4.1f}  {s[:100]}")

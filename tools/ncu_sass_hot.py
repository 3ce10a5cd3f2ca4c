"""Hot-spot view of an ncu SASS source page (development aid):
  ncu -i rep --page source --csv --print-source sass > sass.csv
  python tools/ncu_sass_hot.py sass.csv
Prints the sampled-stall totals, the per-loop totals (innermost backward-branch
loops), every barrier instruction with its samples, and the hottest
instructions with their dominant stall reasons."""
import csv
import re
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
# one section per kernel ("Kernel Name" line, header, rows): take the first
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hi]
data = []
for r in rows[hi + 1:]:
    if r and r[0] in ("Kernel Name", "Address"):
        break
    if len(r) == len(hdr):
        data.append(r)
col = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ins = []
for r in data:
    a = int(r[col["Address"]], 16)
    s = int(r[col["Warp Stall Sampling (All Samples)"]] or 0)
    st = {h: int(r[col[h]] or 0) for h in stalls}
    ex = int(r[col["Instructions Executed"]] or 0)
    ins.append((a, r[col["Source"]].strip(), s, st, ex))
base = ins[0][0]
tot = sum(i[2] for i in ins)
agg = Counter()
for i in ins:
    agg.update(i[3])
print(f"samples {tot}; instructions executed {sum(i[4] for i in ins):.3e}")
print("stalls:", ", ".join(f"{k[6:]} {v / tot:.1%}" for k, v in agg.most_common(10)))
# loops
addr = {a: k for k, (a, *_) in enumerate(ins)}
loops = []
for k, (a, t, *_rest) in enumerate(ins):
    m = re.search(r"BRA\s+(?:`?\(?\.?L?_?x?_?)?(0x[0-9a-f]+)", t)
    if m:
        tgt = int(m.group(1), 16)
        tgt_abs = tgt if tgt in addr else base + tgt
        if tgt_abs < a and tgt_abs in addr:
            loops.append((addr[tgt_abs], k))
print("\nloops (start-end offset, len, samples %, executed, top stalls):")
for s0, s1 in sorted(loops, key=lambda x: x[1] - x[0])[:40]:
    body = ins[s0:s1 + 1]
    sm = sum(b[2] for b in body)
    if sm < 0.01 * tot:
        continue
    c = Counter()
    for b in body:
        c.update(b[3])
    print(f"  {ins[s0][0]-base:#07x}-{ins[s1][0]-base:#07x} {s1-s0+1:5d} {sm/tot:6.1%} "
          f"exec {sum(b[4] for b in body):.2e}  " + ", ".join(f"{k[6:]} {v/sm:.0%}" for k, v in c.most_common(4)))
print("\nbarriers:")
for a, t, s, st, ex in ins:
    if t.startswith("BAR") or "BAR.SYNC" in t or "SYNCS" in t:
        print(f"  {a-base:#07x} {t[:50]:50s} {s/tot:6.2%}  exec {ex}")
print("\nhottest instructions:")
for a, t, s, st, ex in sorted(ins, key=lambda x: -x[2])[:40]:
    top = ", ".join(f"{k[6:]} {v}" for k, v in Counter(st).most_common(2))
    print(f"  {a-base:#07x} {t[:60]:60s} {s/tot:6.2%}  {top}")

# instructions executed per innermost loop (each instruction assigned to the
# shortest loop containing it; the rest is "straight-line")
owner = [None] * len(ins)
for s0, s1 in sorted(loops, key=lambda x: x[1] - x[0], reverse=True):
    for k in range(s0, s1 + 1):
        owner[k] = (s0, s1)
by = Counter()
smp = Counter()
for k, i in enumerate(ins):
    by[owner[k]] += i[4]
    smp[owner[k]] += i[2]
allx = sum(i[4] for i in ins)
print("\ninstructions executed by innermost loop:")
for o, v in by.most_common(16):
    lab = "straight" if o is None else f"{ins[o[0]][0]-base:#07x}-{ins[o[1]][0]-base:#07x} ({o[1]-o[0]+1} instr)"
    print(f"  {lab:32s} {v:.3e} {v/allx:6.1%}  samples {smp[o]/tot:6.1%}")

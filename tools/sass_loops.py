"""Lists backward-branch loops of a kernel in a cubin/object (cuobjdump
-sass) with their instruction counts and opcode histogram (development aid).
usage: python tools/sass_loops.py obj.o kernel_substring [min_len]"""
import re, subprocess, sys
from collections import Counter
obj, name = sys.argv[1], sys.argv[2]
minlen = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
for f in funcs:
    head = f.split("\n", 1)[0]
    if name not in head:
        continue
    ins = []
    for ln in f.split("\n"):
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    addr = {a: i for i, (a, _) in enumerate(ins)}
    print("==", head.strip()[:120], len(ins), "instructions")
    for i, (a, t) in enumerate(ins):
        m = re.search(r"BRA (?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", t)
        mm = re.search(r"BRA\s+0x([0-9a-f]+)", t)
        if mm:
            tgt = int(mm.group(1), 16)
            if tgt < a and tgt in addr and i - addr[tgt] + 1 >= minlen:
                body = ins[addr[tgt]:i + 1]
                ops = Counter(re.sub(r"^@!?U?P\w+\s+", "", x[1]).split()[0].split(".")[0] for x in body)
                print(f"  loop {tgt:#x}-{a:#x}: {len(body)} instr; " +
                      ", ".join(f"{k}:{v}" for k, v in ops.most_common(14)))

"""List the backward-branch loops of a SASS dump with opcode histograms:
    cuobjdump -sass -fun NAME obj.o > k.sass; python tools/sass_loops.py k.sass [min_len]"""
import collections
import re
import sys

lines = open(sys.argv[1]).read().splitlines()
minlen = int(sys.argv[2]) if len(sys.argv) > 2 else 100
ins = []
for ln in lines:
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: i for i, (a, _) in enumerate(ins)}
for i, (a, txt) in enumerate(ins):
    m = re.search(r"BRA(?:\.\w+)?\s+(?:!?U?P\d, )?(0x[0-9a-f]+)", txt)
    if not m:
        continue
    tgt = int(m.group(1), 16)
    if tgt >= a or tgt not in addr:
        continue
    j = addr[tgt]
    body = ins[j:i + 1]
    if len(body) < minlen:
        continue
    h = collections.Counter()
    for _, t in body:
        op = re.sub(r"^@!?U?P\w+\s+", "", t).split()[0]
        h[op] += 1
    fp = sum(v for k, v in h.items() if k.startswith(("FADD", "FMUL", "FFMA")))
    print(f"loop {hex(tgt)}..{hex(a)} len={len(body)} fp32={fp} mufu={h.get('MUFU.RSQ', 0)} other={len(body) - fp - h.get('MUFU.RSQ', 0)}")
    print("   ", ", ".join(f"{k}:{v}" for k, v in h.most_common() if not k.startswith(("FADD", "FMUL", "FFMA", "MUFU"))))

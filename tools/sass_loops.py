"""Summarise the innermost loops of a SASS listing (cuobjdump -sass): instruction mix per loop body.
Usage: python tools/sass_loops.py file.sass"""
import collections
import re
import sys

lines = open(sys.argv[1]).read().splitlines()
ins = []
for ln in lines:
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)(.*?);", ln)
    if m:
        ins.append((int(m.group(1), 16), m.group(3), m.group(4)))
addr = [a for a, _, _ in ins]
for i, (a, op, rest) in enumerate(ins):
    if op.startswith("BRA"):
        t = re.search(r"0x([0-9a-f]+)", rest)
        if t and int(t.group(1), 16) < a:
            lo = int(t.group(1), 16)
            body = [o for (b, o, _) in ins if lo <= b <= a]
            c = collections.Counter(o.split(".")[0] for o in body)
            print(f"loop 0x{lo:x}-0x{a:x}: {len(body)} instrs: " + ", ".join(f"{k} {v}" for k, v in c.most_common()))

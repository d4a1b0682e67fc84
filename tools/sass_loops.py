#!/usr/bin/env python
"""Developer tool: list the loops (backward branches) of a SASS dump made by tools/sass_fn.sh with their static
instruction counts and opcode mix."""
import re, sys, collections
ins = []
for l in open(sys.argv[1]):
    m = re.match(r'\s*/\*([0-9a-f]{4,5})\*/\s+(.*?);', l)
    if m: ins.append((int(m.group(1), 16), m.group(2).strip()))
addr_idx = {a: i for i, (a, _) in enumerate(ins)}
for i, (a, t) in enumerate(ins):
    m = re.search(r'\bBRA(?:\.U)?\s+(?:!?U?P\d+,\s*)?0x([0-9a-f]+)', t)
    if m:
        tgt = int(m.group(1), 16)
        if tgt <= a and tgt in addr_idx:
            body = ins[addr_idx[tgt]:i + 1]
            mix = collections.Counter()
            for _, x in body:
                x = re.sub(r'^@!?U?P\d+\s+', '', x)
                mix[x.split()[0].split('.')[0]] += 1
            print(f"loop {tgt:05x}-{a:05x}: {len(body)} instr  " + " ".join(f"{k}:{v}" for k, v in mix.most_common(12)))

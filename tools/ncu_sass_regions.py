#!/usr/bin/env python
"""Developer tool: per-region instruction budget of a kernel from an ncu source-page export.

    ncu -i prof.ncu-rep --page source --csv --print-source sass > k1_sass.csv
    python tools/ncu_sass_regions.py k1_sass.csv --pairs 8192 --dim 5000 [--dump]

Splits the SASS listing at backward-branch targets / branch instructions into straight-line regions, prints for each
region its static length, executed warp instructions, share, thread-instructions per pair-gene and stall samples, and
(--dump) the hottest instructions. Used for the per-pass instruction table of K1 in profiles/."""
import argparse
import csv
import re
import sys


def load(path):
    rows = []
    with open(path, newline="") as fh:
        rd = csv.reader(fh)
        header = None
        for r in rd:
            if header is None:
                if r and r[0] == "Address":
                    header = r
                continue
            if len(r) < len(header):
                continue
            rows.append(dict(zip(header, r)))
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--pairs", type=int, default=8192)
    ap.add_argument("--dim", type=int, default=5000)
    ap.add_argument("--dump", action="store_true")
    ap.add_argument("--min-share", type=float, default=0.3)
    ap.add_argument("--marks", default="", help="comma-separated region labels by first instruction index: idx=name,...")
    a = ap.parse_args()
    rows = load(a.csv)
    ins = []
    for r in rows:
        ins.append(dict(addr=int(r["Address"], 16), text=r["Source"].strip(), n=int(r["Instructions Executed"] or 0),
                        thr=int(r["Thread Instructions Executed"] or 0), stall=int(r["Warp Stall Sampling (All Samples)"] or 0)))
    base = ins[0]["addr"]
    idx = {i["addr"] - base: k for k, i in enumerate(ins)}
    cuts = {0}
    for k, i in enumerate(ins):
        m = re.search(r"\bBRA(?:\.[A-Z.]+)?\s+(?:!?U?P\d+,\s*)?`?\(?\.?L?_?x?_?\d*\)?|0x([0-9a-f]+)", i["text"])
        if re.search(r"\b(BRA|BSSY|BSYNC|CALL|RET|EXIT|WARPSYNC|BREAK)\b", i["text"]):
            cuts.add(k + 1)
        t = re.search(r"\bBRA\b.*0x([0-9a-f]+)", i["text"])
        if t:
            off = int(t.group(1), 16)
            if off in idx:
                cuts.add(idx[off])
    cuts = sorted(c for c in cuts if c < len(ins))
    total = sum(i["n"] for i in ins)
    total_stall = sum(i["stall"] for i in ins) or 1
    pg = float(a.pairs) * a.dim
    print(f"total warp instructions {total:,}  = {total * 32 / pg:.1f} thread-instr per pair-gene; stall samples {total_stall}")
    print(f"{'first':>6} {'len':>4} {'exec/instr':>12} {'warp instr':>14} {'share%':>7} {'thr/pg':>7} {'stall%':>7}  first instruction")
    regions = []
    for c0, c1 in zip(cuts, cuts[1:] + [len(ins)]):
        seg = ins[c0:c1]
        n = sum(i["n"] for i in seg)
        regions.append((c0, c1, n, sum(i["stall"] for i in seg)))
    for c0, c1, n, st in regions:
        if 100.0 * n / total < a.min_share:
            continue
        seg = ins[c0:c1]
        print(f"{c0:6d} {c1 - c0:4d} {n / (c1 - c0):12.0f} {n:14,} {100.0 * n / total:7.2f} {n * 32 / pg:7.2f} {100.0 * st / total_stall:7.2f}  {seg[0]['text'][:70]}")
    if a.dump:
        print("\n-- instructions with >= 0.5 % of the stall samples or of the executed instructions")
        for k, i in enumerate(ins):
            if i["stall"] >= 0.005 * total_stall or i["n"] >= 0.005 * total:
                print(f"{k:6d} {i['n']:12,} {100.0 * i['stall'] / total_stall:6.2f}%  {i['text'][:100]}")


if __name__ == "__main__":
    main()

"""Attribute ncu per-SASS-instruction counts to source lines.

usage: python tools/sass_attrib.py <ncu sass csv> <nvdisasm --print-line-info dump> <function symbol> [top]
The ncu csv is `ncu -i X.ncu-rep --page source --csv --print-source=sass`; the
dump is `nvdisasm --print-line-info <cubin>` of the SAME build.
"""
import collections
import csv
import re
import sys


def main():
    sass_csv, dump, sym = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    lines = open(dump).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith(".text." + sym + ":")][0]
    loc = {}
    cur = ("?", 0)
    for l in lines[start + 1:]:
        if l.startswith("//----") or l.startswith(".text."):
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
        if m:
            loc[int(m.group(1), 16)] = cur
    rows = list(csv.reader(open(sass_csv)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    by = collections.Counter()
    st = collections.Counter()
    tot = tots = 0.0
    base = None
    for r in rows[2:]:
        try:
            a0 = int(r[ix["Address"]], 16)
        except (ValueError, IndexError):
            continue
        base = a0 if base is None else min(base, a0)
    for r in rows[2:]:
        if len(r) <= ix["Instructions Executed"]:
            continue
        try:
            a = int(r[ix["Address"]], 16) - base
            n = float(r[ix["Instructions Executed"]] or 0)
            s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:
            continue
        k = loc.get(a, ("?", 0))
        by[k] += n
        st[k] += s
        tot += n
        tots += s
    print(f"total instructions {tot:.3e}, stall samples {tots:.0f}")
    for k, n in by.most_common(top):
        print(f"{k[0]:>18s}:{k[1]:<5d} {100 * n / tot:6.2f}% inst {100 * st[k] / max(tots, 1):6.2f}% stall")


if __name__ == "__main__":
    main()

"""Attribute ncu per-SASS instruction counts to source regions through the
inlining chain (nvdisasm --print-line-info-inline).

usage: python tools/sass_attrib_inline.py <ncu sass csv> <nvdisasm -gi dump> <symbol> [depth] [top]
Groups by the chain truncated to `depth` levels counted from the OUTERMOST
frame (the kernel body), so depth 2 splits run_sim's statements etc.
"""
import collections
import csv
import re
import sys


def main():
    sass_csv, dump, sym = sys.argv[1:4]
    depth = int(sys.argv[4]) if len(sys.argv) > 4 else 2
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
    lines = open(dump).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith(".text." + sym + ":")][0]
    loc, cur = {}, ()
    for l in lines[start + 1:]:
        if l.startswith("//----") or l.startswith(".text."):
            break
        if "//## File" in l:
            parts = re.findall(r'"([^"]+)", line (\d+)', l)
            cur = tuple((f.split("/")[-1], int(n)) for f, n in parts)  # innermost first
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
        if m:
            loc[int(m.group(1), 16)] = cur
    rows = list(csv.reader(open(sass_csv)))
    ix = {h: i for i, h in enumerate(rows[1])}
    data = []
    for r in rows[2:]:
        try:
            data.append((int(r[ix["Address"]], 16), float(r[ix["Instructions Executed"]] or 0),
                         float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)))
        except (ValueError, IndexError):
            pass
    base = min(a for a, _, _ in data)
    by, st = collections.Counter(), collections.Counter()
    tot = tots = 0.0
    for a, n, s in data:
        chain = loc.get(a - base, ())
        key = tuple(reversed(chain))[:depth]
        by[key] += n
        st[key] += s
        tot += n
        tots += s
    print(f"total {tot:.3e} inst")
    for k, n in by.most_common(top):
        print(f"{100 * n / tot:6.2f}% inst {100 * st[k] / max(tots, 1):6.2f}% stall  " +
              " > ".join(f"{f}:{l}" for f, l in k))


if __name__ == "__main__":
    main()

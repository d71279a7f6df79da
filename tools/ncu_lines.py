#!/usr/bin/env python
"""Per-source-line instruction counts and warp-stall reasons from an
`ncu --page source --csv --print-source cuda,sass` export (development aid)."""
import collections
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr = fn = last = None
    instr = collections.Counter()
    stalls = collections.defaultdict(collections.Counter)
    tot_st = collections.Counter()
    src = {}
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fn = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            ie = hdr.index("Instructions Executed")
            sidx = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        line = r[0] if r[0] else last
        last = line
        key = (fn, line)
        if r[1]:
            src[key] = r[1].strip()[:80]
        if r[0]:
            continue  # source row: the SASS rows below carry the counters
        try:
            instr[key] += float(r[ie] or 0)
        except ValueError:
            pass
        for i in sidx:
            try:
                v = float(r[i] or 0)
            except ValueError:
                v = 0.0
            stalls[key][hdr[i][6:]] += v
            tot_st[hdr[i][6:]] += v
    ti = sum(instr.values())
    ts = sum(tot_st.values())
    print(f"instructions {ti:.0f}; stall samples {ts:.0f}")
    print("  " + ", ".join(f"{k}:{v / ts * 100:.1f}%" for k, v in tot_st.most_common(8)))
    keys = sorted(set(instr) | set(stalls), key=lambda k: -sum(stalls[k].values()))
    for k in keys[:top]:
        s = sum(stalls[k].values())
        t3 = ", ".join(f"{a}:{b / max(s, 1) * 100:.0f}%" for a, b in stalls[k].most_common(3))
        print(f"{s / ts * 100:5.1f}% smp {instr[k] / ti * 100:5.1f}% ins  {k[0]}:{k[1]} [{t3}] {src.get(k, '')}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)

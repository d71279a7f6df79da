#!/usr/bin/env python
"""Aggregate warp-stall samples of an `ncu --page source --csv --print-source cuda,sass` export by
CUDA source line (and optionally print the top SASS instructions)."""
import csv
import sys
from collections import defaultdict


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    cur_file = None
    header = None
    by_line = defaultdict(lambda: [0, 0, ""])
    total = 0
    sass_top = []
    last_line = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            continue
        if r[0] == "Line No":
            header = r
            idx_all = header.index("Warp Stall Sampling (All Samples)")
            idx_ni = header.index("Warp Stall Sampling (Not-issued Samples)")
            continue
        if header is None:
            continue
        try:
            s_all = int(r[idx_all] or 0)
            s_ni = int(r[idx_ni] or 0)
        except (ValueError, IndexError):
            continue
        line = r[0] if r[0] else last_line
        last_line = line
        key = (cur_file, line)
        by_line[key][0] += s_all
        by_line[key][1] += s_ni
        if r[1]:
            by_line[key][2] = r[1].strip()[:110]
        total += s_all
        sass_top.append((s_all, cur_file, line, r[3][:90] if len(r) > 3 else ""))
    print(f"total samples {total}")
    for (f, ln), (a, ni, src) in sorted(by_line.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100.0 * a / max(total, 1):6.2f}%  {f}:{ln:>5}  {src}")
    print("--- top SASS")
    for a, f, ln, s in sorted(sass_top, key=lambda t: -t[0])[:25]:
        print(f"{100.0 * a / max(total, 1):6.2f}%  {f}:{ln}  {s}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)

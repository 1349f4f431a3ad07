"""Aggregate ncu warp-stall samples by CUDA source line from a
`ncu -i rep --page source --csv --print-source cuda,sass` export.

    python tools/ncu_lines.py export.csv [top]
"""
import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    agg = defaultdict(float)
    text = {}
    fname = None
    hdr = None
    cur = None
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            i_s = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        if r[0] not in ("", "-"):
            cur = (fname, r[0])
            text[cur] = r[1]
        if r[2] not in ("", "-") and cur is not None:  # a SASS row under the current line
            try:
                agg[cur] += float(r[i_s] or 0)
            except ValueError:
                pass
    tot = sum(agg.values()) or 1.0
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{100 * v / tot:6.2f}%  {k[0]}:{k[1]:>5}  {text[k][:90]}")


if __name__ == "__main__":
    main()

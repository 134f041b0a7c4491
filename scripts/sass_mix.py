"""Per-opcode executed warp instructions and stall samples from an ncu
source page (--page source --csv --print-source sass)."""
import csv
import sys
from collections import Counter


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ci, si, xi = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    ex, st = Counter(), Counter()
    for r in rows[2:]:
        if len(r) <= max(xi, si):
            continue
        op = r[ci].strip().split()
        if not op:
            continue
        o = op[0]
        if o.startswith("@"):
            o = op[1] if len(op) > 1 else o
        o = o.split(".")[0]
        try:
            ex[o] += int(float(r[si] or 0))
            st[o] += int(float(r[xi] or 0))
        except ValueError:                 # a repeated header row
            continue
    tot = sum(ex.values())
    tots = sum(st.values())
    print(f"total warp instructions {tot}, stall samples {tots}")
    for o, n in ex.most_common(top):
        print(f"{o:12s} {n:12d} {100*n/tot:5.1f}%   stalls {100*st[o]/max(tots,1):5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])

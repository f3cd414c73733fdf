"""Summarise an `ncu --page source --csv --print-source sass` export: instruction
mix and stall samples by opcode, plus the hottest SASS lines (run here, no GPU)."""
import csv
import sys
from collections import Counter


def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hi]
    ie, ss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    data = [r for r in rows[hi + 1:] if len(r) > ie and r[ie].replace(".", "", 1).isdigit()]
    return data, ie, ss


def main(path, top=25):
    data, ie, ss = load(path)
    tot = sum(float(r[ie]) for r in data)
    tots = sum(float(r[ss] or 0) for r in data) or 1
    print("warp instructions %.4g, stall samples %d, SASS lines %d" % (tot, tots, len(data)))
    c, cs = Counter(), Counter()
    for r in data:
        toks = r[1].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        op = op.split(".")[0]
        c[op] += float(r[ie])
        cs[op] += float(r[ss] or 0)
    for k, v in c.most_common(top):
        print("%-10s %10.4g  %5.1f%% inst  %5.1f%% stalls" % (k, v, 100 * v / tot, 100 * cs[k] / tots))
    print("--- hottest lines by stall samples")
    for r in sorted(data, key=lambda r: -float(r[ss] or 0))[:top]:
        print(r[0][-5:], "%-60s" % r[1].strip()[:60], r[ie], r[ss])


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)

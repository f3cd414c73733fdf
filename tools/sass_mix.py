"""Dynamic instruction mix of one kernel from an ncu `--page source --csv
--print-source sass` export: executed warp instructions per opcode, the
hottest straight-line blocks, and per-output counts (pass outputs=N)."""
import csv
import sys
from collections import Counter


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ia, isrc, iex, ist = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), \
        hdr.index("Warp Stall Sampling (All Samples)")
    out = []
    for r in rows[2:]:
        if len(r) <= iex:
            continue
        try:
            out.append((int(r[ia], 16), r[isrc].strip(), int(r[iex] or 0), int(r[ist] or 0)))
        except ValueError:
            continue
    return out


def main(path, outputs=0):
    ins = load(path)
    tot = sum(x[2] for x in ins)
    ops = Counter()
    for a, s, n, st in ins:
        op = s.split()[0] if s else "?"
        if op.startswith("@"):
            op = s.split()[1]
        ops[op.split(".")[0]] += n
    print(f"total warp instructions {tot:,}" + (f"  per output (thread-instr) {32 * tot / outputs:.1f}" if outputs else ""))
    for op, n in ops.most_common(25):
        print(f"  {op:10s} {n:14,} {100 * n / tot:5.1f}%")
    # hottest instructions by stall samples
    print("top stall-sampled instructions:")
    for a, s, n, st in sorted(ins, key=lambda x: -x[3])[:25]:
        print(f"  {a & 0xFFFFF:06x} samples {st:6d} exec {n:10,}  {s[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)

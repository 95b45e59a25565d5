"""Summarise an ncu `--page source --print-source sass --csv` export: executed
instructions and stall samples per opcode, plus the hottest instructions."""
import collections
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    ops = collections.Counter()
    stalls = collections.Counter()
    samples = []
    total = 0
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        src = r[ix["Source"]].strip()
        try:
            ex = int(r[ix["Instructions Executed"]] or 0)
            smp = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:
            continue
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        ops[op] += ex
        stalls[op] += smp
        total += ex
        samples.append((smp, ex, r[ix["Address"]], src[:90]))
    print(f"total executed warp-instructions: {total}")
    print("opcode           executed    share   stall-samples")
    ts = sum(stalls.values()) or 1
    for op, ex in ops.most_common(30):
        print(f"{op:14s} {ex:12d} {100*ex/total:7.2f}% {100*stalls[op]/ts:7.2f}%")
    print("\nhottest instructions by stall samples:")
    for smp, ex, addr, src in sorted(samples, reverse=True)[:top]:
        print(f"{smp:8d} {ex:10d} {addr} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)

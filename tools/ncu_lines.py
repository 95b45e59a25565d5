"""Per-source-line executed instructions and stall samples from
`ncu --page source --print-source cuda,sass --csv` (lines with metrics)."""
import csv
import subprocess
import sys


def main(path, top=45):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    ix = {h: i for i, h in enumerate(hdr) if h not in ("Source",)}
    ex_i = hdr.index("Instructions Executed")
    st_i = hdr.index("Warp Stall Sampling (All Samples)")
    lines = []
    tot_ex = tot_st = 0
    for r in rows:
        if len(r) <= ex_i or not r[0] or not r[0].isdigit():
            continue
        try:
            ex, st = int(r[ex_i] or 0), int(r[st_i] or 0)
        except ValueError:
            continue
        tot_ex += ex
        tot_st += st
        lines.append((ex, st, int(r[0]), r[1][:90]))
    print(f"total executed {tot_ex}  stall samples {tot_st}")
    for ex, st, ln, src in sorted(lines, reverse=True)[:top]:
        print(f"{100*ex/tot_ex:6.2f}% ex {100*st/max(tot_st,1):6.2f}% st  L{ln:4d} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 45)

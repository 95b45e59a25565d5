"""Print the headline metrics of an ncu report (details page)."""
import csv
import subprocess
import sys

KEEP = ["Duration", "Executed Ipc Active", "Issue Slots Busy", "Active Warps Per Scheduler",
        "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "Executed Instructions",
        "Registers Per Thread", "Achieved Active Warps Per SM", "DRAM Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block",
        "Theoretical Occupancy", "Achieved Occupancy"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    ix = {h: i for i, h in enumerate(rows[0])}
    for r in rows[1:]:
        if r[ix["Metric Name"]] in KEEP:
            print(f"{r[ix['Kernel Name']][:40]:40s} {r[ix['Metric Name']]:40s} {r[ix['Metric Unit']]:12s} {r[ix['Metric Value']]}")


if __name__ == "__main__":
    main(sys.argv[1])

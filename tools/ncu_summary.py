"""Print selected metrics of each kernel in an .ncu-rep (details page)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
keys = sys.argv[2].split(",") if len(sys.argv) > 2 else [
    "Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
    "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Issue Slots Busy",
    "No Eligible", "Dynamic Shared Memory Per Block", "Static Shared Memory Per Block"]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
ki, ni, mi, vi, ui = (h.index(c) for c in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
cur = None
for r in rows[1:]:
    if r[ki] != cur:
        cur = r[ki]
        print(f"[{cur}] {r[ni][:100]}")
    if any(k in r[mi] for k in keys):
        print(f"    {r[mi]:45s} {r[vi]:>14s} {r[ui]}")

"""Hot SASS lines of an ncu report: python tools/ncu_hot.py <rep> [n]
Prints stall samples / executed count per instruction, top n, and the mbarrier
spin loops (SYNCS try-wait) with their smem offsets."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[1]
data = rows[2:]
iS = h.index("Warp Stall Sampling (All Samples)")
iE = h.index("Instructions Executed")
iSrc = h.index("Source")
tot = sum(int(r[iS] or 0) for r in data)
print("samples", tot, "instructions", sum(int(r[iE] or 0) for r in data))
for r in sorted(data, key=lambda r: -int(r[iS] or 0))[:n]:
    print(f"{int(r[iS]):6d} {int(r[iE] or 0):9d} {r[0][-5:]} {r[iSrc][:100]}")
print("--- spin loops")
for r in data:
    if "TRYWAIT" in r[iSrc] and int(r[iE] or 0) > 1000:
        print(f"{int(r[iE]):9d} {r[0][-5:]} {r[iSrc][:100]}")

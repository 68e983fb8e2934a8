"""Instructions executed / stall samples per CUDA source line of an ncu report:
python tools/ncu_lines.py <rep> [n] -> top n lines (needs -lineinfo builds)."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
inst = collections.Counter()
samp = collections.Counter()
src = {}
fname = ""
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < len(hdr) or not r[0].isdigit():
        continue
    key = (fname, int(r[0]))
    src[key] = r[1].strip()
    try:
        inst[key] += int(r[hdr.index("Instructions Executed")] or 0)
        samp[key] += int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError:
        pass
tot_i, tot_s = sum(inst.values()), sum(samp.values())
print(f"instructions {tot_i}  samples {tot_s}")
for key, v in inst.most_common(n):
    print(f"{v:10d} {100 * v / max(tot_i, 1):5.1f}% {samp[key]:6d} {key[0]}:{key[1]:4d} {src[key][:90]}")

"""Summarise gpurun_out/ ncu artefacts into profiles/ (tracked).

  python tools/summarize_profiles.py <round-tag> [launches.csv] [prof.ncu-rep ...]

* launch list (``ncu --metrics gpu__time_duration.sum``): per-kernel totals of
  the LAST network forward in the capture (from the last stem launch on), with
  each kernel's share of that forward -> profiles/<tag>_launches.txt;
* ``--set full`` reports: key counters per captured launch
  -> profiles/<tag>_ncu_<name>.txt.
"""
import collections
import csv
import io
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sectors.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "sm__cycles_elapsed.avg.per_second",
]


def launches(path: Path, start_pattern: str = "stem"):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    starts = [i for i, d in enumerate(data) if start_pattern in d["Kernel Name"]]
    last = data[starts[-1]:] if starts else data
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    agg = collections.defaultdict(lambda: [0, 0.0])
    seq = []
    for d in last:
        us = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1e-3)
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += us
        seq.append((us, d["Grid Size"], name))
    tot = sum(v[1] for v in agg.values())
    out = io.StringIO()
    out.write(f"# one forward from the last '{start_pattern}' launch: {len(last)} launches, "
              f"{tot:.1f} us serialised (ncu, cold cache: compare shares)\n")
    out.write(f"{'us':>10} {'share':>6} {'n':>4}  kernel\n")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.write(f"{t:10.1f} {100 * t / tot:5.1f}% {c:4d}  {k}\n")
    out.write("\n# launch sequence (us, grid, kernel)\n")
    for us, g, nm in seq:
        out.write(f"{us:9.1f} {g:>14} {nm}\n")
    return out.getvalue()


def ncu_full(rep: Path):
    r = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(r.stdout)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out = io.StringIO()
    for i, d in enumerate(data):
        out.write(f"## launch {i}: {d[hdr.index('Kernel Name')][:90]} grid {d[hdr.index('Grid Size')]} "
                  f"block {d[hdr.index('Block Size')]}\n")
        for k in KEYS:
            if k in hdr:
                j = hdr.index(k)
                out.write(f"  {k:70s} {d[j]:>14} {units[j]}\n")
    return out.getvalue()


def main():
    tag = sys.argv[1]
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    for a in sys.argv[2:]:
        p = Path(a)
        if p.suffix == ".csv":
            (prof / f"{tag}_launches.txt").write_text(launches(p))
        elif p.suffix == ".ncu-rep":
            (prof / f"{tag}_ncu_{p.stem}.txt").write_text(ncu_full(p))


if __name__ == "__main__":
    main()

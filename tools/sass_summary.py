"""Per-kernel SASS instruction-class counts of the built library (north-star
evidence: tcgen05 / TMA / TMEM instructions per instantiation).

  python tools/sass_summary.py [out.txt]      (default profiles/sass_summary.txt)

Reads ``cuobjdump -sass`` of paper_2308_15949_b200/_laud.so and writes, per
function (demangled), the static counts of the Blackwell-native classes:
UTCHMMA (tcgen05.mma, .2CTA = cta_group::2), UTCBAR (tcgen05.commit),
UTMALDG (TMA loads, incl. .GATHER4 / 2D / 3D / 4D), UBLKCP (bulk copies),
LDTM / STTM (tcgen05.ld / st), SYNCS (mbarrier), plus legacy HMMA (must be 0)
and LDGSTS (cp.async), and the total instruction count.  The hot kernels' full
SASS is written next to it (profiles/sass_<kernel>.txt).
"""
import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
SO = ROOT / "paper_2308_15949_b200" / "_laud.so"
CLASSES = ["UTCHMMA", "UTCHMMA.2CTA", "UTCBAR", "UTMALDG.2D", "UTMALDG.2D.GATHER4", "UTMALDG.3D", "UTMALDG.4D",
           "UBLKCP", "LDTM", "STTM", "UTCATOMSWS", "SYNCS", "HMMA", "LDGSTS", "STG", "LDG"]
HOT = {"patch_conv_kernel<2, 128>": "sass_patch_conv_s2.txt",
       "conv_gemm_kernel<256, 3, 1, false, 0, 6>": "sass_conv_gemm_conv3.txt"}


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return r.stdout.splitlines()


def main(out):
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", str(SO)], capture_output=True,
                          text=True).stdout
    funcs = []
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = [m.group(1), []]
            funcs.append(cur)
        elif cur is not None and re.match(r"\s*/\*[0-9a-f]{4,}\*/", line):
            cur[1].append(line)
    names = demangle([f[0] for f in funcs])
    rows = []
    for (mangled, body), name in zip(funcs, names):
        c = collections.Counter()
        for ln in body:
            ins = re.sub(r"^\s*/\*[0-9a-f]+\*/\s*", "", ln).split(";")[0].strip()
            ins = re.sub(r"^@!?U?P\w+\s+", "", ins)
            op = ins.split(" ")[0] if ins else ""
            fam = ("SYNCS", "LDTM", "STTM", "LDGSTS", "STG", "LDG", "HMMA", "UBLKCP", "UTCBAR", "UTCATOMSWS")
            for k in CLASSES:
                if op == k or (k in fam and op.startswith(k + ".")):
                    c[k] += 1
            if op.startswith("UTCHMMA") and "2CTA" in op:
                c["UTCHMMA.2CTA"] += 1
        short = name.replace("void ", "").split("(")[0].replace("laud::", "")
        rows.append((short, len(body), c))
        for key, fn in HOT.items():
            if key.replace(" ", "") in short.replace(" ", "").replace("(bool)", "").replace("(int)", ""):
                (ROOT / "profiles" / fn).write_text(f"// {name}\n" + "\n".join(body) + "\n")
    with open(out, "w") as f:
        f.write("# static SASS instruction classes per kernel of _laud.so (cuobjdump -sass; "
                "tools/sass_summary.py)\n")
        f.write(f"{'instrs':>7} " + " ".join(f"{k:>8}" for k in CLASSES) + "  kernel\n")
        for short, n, c in sorted(rows, key=lambda r: r[0]):
            f.write(f"{n:7d} " + " ".join(f"{c.get(k, 0):8d}" for k in CLASSES) + f"  {short}\n")
    print(out)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else ROOT / "profiles" / "sass_summary.txt")

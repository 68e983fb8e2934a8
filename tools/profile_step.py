"""Per-launch table of one eager LAUD network forward (CUDA events via laud_profile_*)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_15949_b200 import _lib
from paper_2308_15949_b200.network import LaudNetwork, random_images

arch = sys.argv[1] if len(sys.argv) > 1 else "resnet101"
para = sys.argv[2] if len(sys.argv) > 2 else "spatial"
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 256
net = LaudNetwork(arch, para, sys.argv[4] if len(sys.argv) > 4 else ("4-4-2-1" if arch.startswith("regnet") else "4-2-2-1"), 0.5)
img = random_images(batch)
net.calibrate(img)
for _ in range(3):
    net.forward(img)
torch.cuda.synchronize()
lib = _lib.lib()
lib.laud_profile_begin()
net.forward(img)
recs = (_lib.ProfileRecord * 4096)()
n = lib.laud_profile_end(recs, 4096)
tot = sum(r.ms for r in recs[:n])
rows = []
for i, r in enumerate(recs[:n]):
    fl = 2.0 * r.rows * r.n_out * r.k
    tf = fl / (r.ms * 1e-3) / 1e12 if r.ms else 0
    # rough compulsory bytes of a conv: A rows*k*2 (k counts taps) / taps... report GB/s of (rows*(k_in+n_out)*2)
    rows.append(dict(i=i, tag=r.tag, us=round(r.ms * 1e3, 1), rows=r.rows, n_out=r.n_out, k=r.k,
                     tflops=round(tf, 1), bytes=r.bytes))
for d in rows:
    print(json.dumps(d))
print("total_ms", round(tot, 3), "launches", n)

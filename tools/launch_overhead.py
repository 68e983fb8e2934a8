"""Per-launch fixed cost of the conv engine inside a CUDA graph: G back-to-back
tiny convs (one 128x256 tile, K=64) replayed as one graph, with and without PDL."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2308_15949_b200 import channel as CH  # noqa: E402
from paper_2308_15949_b200 import device as D  # noqa: E402


def main():
    torch.cuda.set_device(0)
    m, n, k = int(sys.argv[1]) if len(sys.argv) > 1 else 128, 256, 64
    a = torch.randn(m, k, device="cuda").bfloat16()
    w = D.pack_weight(torch.randn(n, k, 1, 1) * 0.1, k)
    outs = [torch.empty(m, n, device="cuda").bfloat16() for _ in range(2)]
    G = 50

    def seq():
        for i in range(G):
            CH.conv(act=a, in_hw=(m, 1), in_c=k, in_ld=k, weight=w, n_out=n, out=outs[i & 1], out_ld=n,
                    out_hw=(m, 1), batch=1, a_compact=1, relu=1)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        seq()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        seq()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        g.replay()
    e1.record()
    e1.synchronize()
    print(f"rows={m}: {e0.elapsed_time(e1) * 1e3 / (10 * G):.2f} us per launch "
          f"(PDL={os.environ.get('LAUD_PDL', '1')})")


if __name__ == "__main__":
    main()

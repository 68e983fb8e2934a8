"""HBM read / write / copy bandwidth with torch ops (CUDA events, best of 10):
the practical floors the streaming convs are compared against."""
import json
import torch

torch.cuda.set_device(0)
n = 1 << 29  # 1 GiB of bf16
a = torch.empty(n, dtype=torch.bfloat16, device="cuda").normal_()
b = torch.empty_like(a)


def best(fn, byts):
    ts = []
    for _ in range(12):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = min(ts[2:])
    return round(byts / t / 1e6, 1)


out = {
    "write_fill_gbs": best(lambda: b.fill_(1.0), 2 * n),
    "read_sum_gbs": best(lambda: a.sum(), 2 * n),
    "copy_gbs": best(lambda: b.copy_(a), 4 * n),
    "add_3op_gbs": best(lambda: torch.add(a[: n // 2], a[n // 2:], out=b[: n // 2]), 3 * n),
}
print(json.dumps(out))

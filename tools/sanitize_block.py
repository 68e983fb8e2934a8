"""Small spatial / channel / layer / static block forwards for compute-sanitizer
(memcheck, racecheck, synccheck): python tools/sanitize_block.py

Round 2 adds: the small-grid cluster split-K of the halo conv2 (latency_split),
the masker forked onto a second stream, the grouped halo conv2 (RegNet), the
gathered-weight channel schedule (LAUD_CH_GATHER=1), both fused stems and the
split SE FC kernels, the GEMM engine's small-grid split-K (batch-1 static / S = 1 blocks)
and the TMA-store epilogue."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2308_15949_b200 import device as D
from paper_2308_15949_b200.network import make_params


def main():
    torch.cuda.set_device(0)
    for arch, stage, index, s in (("resnet50", 3, 1, 2), ("resnet50", 2, 0, 2), ("resnet50", 1, 1, 4),
                                  ("resnet50", 4, 1, 1), ("regnety-1.6gf", 3, 1, 2)):
        bp = [b for b in make_params(arch, 0)["blocks"] if b["stage"] == stage and b["index"] == index][0]
        blk = bp["block"]
        ep = D.Epilogue(s1=bp["s1"], b1=bp["b1"], relu1=True, s2=bp["s2"], b2=bp["b2"], relu2=True,
                        s3=bp["s3"], b3=bp["b3"], sd=bp["sd"], bd=bp["bd"], relu_out=True)
        db = D.DeviceBlock(blk, bp["w1"], bp["w2"], bp["w3"], bp["wd"], ep, masker_w=bp["masker_w"],
                           fold_scale=True)
        if "se_w1" in bp:
            db.set_se(bp["se_w1"], bp["se_b1"], bp["se_w2"], bp["se_b2"])
        n, h = 2, blk.input_shape.height
        x = torch.randn(n, h, h, db.cin_p, device="cuda").relu_().bfloat16()
        for dense in (False, True):
            db.forward(x.clone(), "spatial", s, conv1_dense=dense)
        aux = torch.cuda.Stream()
        db.forward(x[:1].clone(), "spatial", s, conv1_dense=True, aux_stream=aux, latency_split=True)
        db.forward(x[:1].clone(), "static", latency_split=True)  # GEMM-engine split-K (small grids)
        db.forward(x.clone(), "static")
        db.forward(x.clone(), "layer", coarse=torch.tensor([1, 0], dtype=torch.uint8, device="cuda"))
        db.enable_grouped_channel()  # EXT for grouped conv2 (no-op otherwise)
        cm = torch.zeros(n * db.cmid_p, dtype=torch.uint8, device="cuda")
        cm[: blk.conv2.out_channels // 2] = 1
        db.forward(x.clone(), "channel", chmask=cm)  # per-sample dynamic width (n < 8)
        n8 = 8  # dense-masked channel schedule (n >= 8)
        x8 = torch.randn(n8, h, h, db.cin_p, device="cuda").relu_().bfloat16()
        cm8 = torch.zeros(n8 * db.cmid_p, dtype=torch.uint8, device="cuda")
        cm8[::3] = 1
        db.forward(x8, "channel", chmask=cm8)
        if blk.conv2.groups == 1:
            os.environ["LAUD_CH_GATHER"] = "1"  # gathered-weight schedule (read per call)
            db.forward(x8, "channel", chmask=cm8)
            os.environ["LAUD_CH_GATHER"] = "0"
        torch.cuda.synchronize()
        print("ok", arch, stage, index, flush=True)
    # fused stems (ResNet 7x7/2 + pool, RegNet 3x3/2) through the network glue
    from paper_2308_15949_b200.network import LaudNetwork
    for arch in ("resnet50", "regnety-1.6gf"):
        net = LaudNetwork(arch, "spatial", "4-4-2-1", 0.5, seed=0)
        img = torch.randint(0, 256, (2, 224, 224, 3), dtype=torch.uint8, device="cuda")
        net.forward(img)
        torch.cuda.synchronize()
        print("ok network", arch, flush=True)


if __name__ == "__main__":
    main()

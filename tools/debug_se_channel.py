import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import laud_oracle as O
from paper_2308_15949_b200 import device as D
from paper_2308_15949_b200.network import make_params
from paper_2308_15949_b200.core import DynamicConfig, Paradigm
bp = [b for b in make_params("regnety-1.6gf", 0)["blocks"] if b["stage"] == 3 and b["index"] == 1][0]
blk = bp["block"]
for use_se in (False, True):
    ep = D.Epilogue(b1=bp["b1"], relu1=True, b2=bp["b2"], relu2=True, b3=bp["b3"], bd=bp["bd"], relu_out=True)
    db = D.DeviceBlock(blk, bp["w1"], bp["w2"], bp["w3"], bp["wd"], ep, grouped_channel_ext=True)
    if use_se:
        db.set_se(bp["se_w1"], bp["se_b1"], bp["se_w2"], bp["se_b2"])
    rng = np.random.default_rng(3)
    n = 3
    ci = blk.input_shape
    x = np.maximum(rng.standard_normal((n, ci.channels, ci.height, ci.width)), 0)
    cm = blk.conv2.out_channels
    cmask = rng.random((n, cm)) < 0.5
    cmask[1] = False
    mm = np.zeros((n, db.cmid_p), np.uint8); mm[:, :cm] = cmask
    y, *_ = db.forward(D.to_device_nhwc(x), "channel", chmask=torch.from_numpy(mm.reshape(-1)).cuda())
    torch.cuda.synchronize()
    yg = D.from_device_nhwc(y, blk.output_shape.channels)
    oep = O.Epilogues(b1=bp["b1"], relu1=True, b2=bp["b2"], relu2=True, b3=bp["b3"], bd=bp["bd"], relu_out=True,
                      **({} if not use_se else dict(se_w1=bp["se_w1"], se_b1=bp["se_b1"], se_w2=bp["se_w2"], se_b2=bp["se_b2"])))
    emu = O.block_forward_sparse(x, O.BlockWeights(bp["w1"], bp["w2"], bp["w3"], bp["wd"]), blk,
                                 DynamicConfig(Paradigm.CHANNEL, channel_granularity=1), O.ChannelMask(cmask, cmask, 1),
                                 epilogues=oep, emulate_bf16=True, grouped_channel_ext=True)
    print("se", use_se, [float(np.linalg.norm(yg[i] - emu[i]) / np.linalg.norm(emu[i])) for i in range(n)])

"""LAUDNet network executor on the CUDA path.

Runs a whole LAUD-ResNet / RegNet-style backbone from the zoo specs:
stem (im2col + tcgen05 GEMM, folded BN, ReLU) -> 3x3/s2 max-pool -> the
bottleneck blocks (spatial / layer / static paradigms, masker-driven masks)
-> global average pool -> FC (fp32 logits).  Everything after the input
upload is stream-ordered on the device with no host synchronisation, so a
forward can be captured in a CUDA graph.

Weights are random-init (no checkpoints exist); folded-BN
scale/bias are synthetic.  Masker weights are random N(0, 1/C); a per-block
masker bias (EXT, a conv bias on the masker's logit 0) is calibrated on a
calibration batch so the block's activation ratio hits ``target_ratio`` —
the role a trained masker's FLOPs loss plays in the paper.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from . import channel as CH
from . import device as D
from .core import Paradigm
from .zoo import build_network, parse_plan

IMAGENET_MEAN = (123.675, 116.28, 103.53)
IMAGENET_STD = (58.395, 57.12, 57.375)


def make_params(arch: str = "resnet101", seed: int = 0) -> dict:
    """Random-init parameters of a whole network, pure numpy (host-side init).

    Shared by the CUDA executor and the CPU oracle's network composer so both
    run the same weights.  Conv weights N(0,1)/sqrt(fan_in) as in
    `reference.py:271-286`; folded BN: scale sqrt(2) after the ReLU'd convs,
    0.5 on conv3, small random biases; masker W ~ N(0, 1/C) of shape (2, C, 1, 1).
    """
    net = build_network(arch)
    rng = np.random.default_rng(seed)
    st = net.stem
    p = {"arch": arch, "net": net}
    p["stem_w"] = rng.standard_normal((st.out_channels, 3, st.kernel, st.kernel)) * \
        np.sqrt(2.0 / (3 * st.kernel ** 2))
    p["stem_b"] = rng.standard_normal(st.out_channels) * 0.01
    blocks = []
    for bi in net.blocks:
        blk = bi.block
        cm, co, ci = blk.conv1.out_channels, blk.conv3.out_channels, blk.input_shape.channels

        def draw(layer):
            cig = layer.in_channels // layer.groups
            return rng.standard_normal((layer.out_channels, cig, layer.kernel, layer.kernel)) / \
                np.sqrt(cig * layer.kernel ** 2)

        wd = rng.standard_normal((co, ci, 1, 1)) / np.sqrt(ci) if blk.has_downsample else None
        w1, w2, w3 = draw(blk.conv1), draw(blk.conv2), draw(blk.conv3)
        blocks.append(dict(
            stage=bi.stage, index=bi.index, block=blk, w1=w1, w2=w2, w3=w3, wd=wd,
            s1=np.full(cm, np.sqrt(2.0)), b1=rng.standard_normal(cm) * 0.05,
            s2=np.full(cm, np.sqrt(2.0)), b2=rng.standard_normal(cm) * 0.05,
            s3=np.full(co, 0.5), b3=rng.standard_normal(co) * 0.05,
            sd=np.ones(co), bd=np.zeros(co),
            masker_w=rng.standard_normal((2, ci, 1, 1)) / np.sqrt(ci)))
        if blk.se_reduction:  # RegNetY squeeze-excitation (EXT; `core.py:195` se_hidden)
            hs = blk.se_hidden
            blocks[-1].update(se_w1=rng.standard_normal((hs, cm)) / np.sqrt(cm),
                              se_b1=rng.standard_normal(hs) * 0.05,
                              se_w2=rng.standard_normal((cm, hs)) / np.sqrt(hs),
                              se_b2=rng.standard_normal(cm) * 0.05 + 1.0)
    p["blocks"] = blocks
    fc_in = net.classifier_features
    p["fc_w"] = rng.standard_normal((net.num_classes, fc_in)) / np.sqrt(fc_in)
    p["fc_b"] = rng.standard_normal(net.num_classes) * 0.01
    return p


@dataclass
class BlockSlot:
    stage: int
    index: int
    db: D.DeviceBlock
    s: int           # spatial granularity (output grid); 0 for static
    fused_in: bool = False  # masker reads the previous block's conv3 dots


class LaudNetwork:
    """A LAUD backbone + classifier resident on one GPU."""

    def __init__(self, arch: str = "resnet101", paradigm: str = "spatial", plan: str = "4-2-2-1",
                 target_ratio: float = 0.5, seed: int = 0, device="cuda"):
        D.require_cuda()
        params = make_params(arch, seed)
        self.params = params
        self.net = params["net"]
        if paradigm == "channel":
            add_channel_maskers(params, parse_plan(plan, self.net, Paradigm.CHANNEL).values, seed)
        self.paradigm = paradigm
        self.target_ratio = target_ratio
        self.device = torch.device(device)
        net = self.net
        para = Paradigm(paradigm)
        if para is Paradigm.SPATIAL or para is Paradigm.CHANNEL:
            self.plan = parse_plan(plan, net, para).values  # S (spatial) or G (channel) per stage
        else:
            self.plan = tuple(net.stage_feature(i + 1).height for i in range(len(net.stages)))
        # stem: k x k / s2 conv over 3 channels via im2col (K = k*k*3 padded to 8)
        st = net.stem
        self.stem_k, self.stem_stride = st.kernel, st.stride
        # im2col K layout per kernel row: ky * seg + kx * 3 + c, seg = pad8(3k)
        seg = D.pad8(st.kernel * 3)
        self.stem_cols = st.kernel * seg
        ws = params["stem_w"]  # (co, 3, k, k)
        wcol = np.zeros((st.out_channels, st.kernel, seg))
        wcol[:, :, : st.kernel * 3] = ws.transpose(0, 2, 3, 1).reshape(st.out_channels, st.kernel, -1)
        wcol = wcol.reshape(st.out_channels, 1, 1, self.stem_cols)
        self.stem_w = D.pack_weight(wcol.transpose(0, 3, 1, 2), self.stem_cols, device)
        self.stem_c = D.pad8(st.out_channels)
        # fused 7x7/2 stem + max-pool (laud_stem_pool): weights [64][ky*32 + kx*4 + c]
        self.stem_fused = (st.kernel == 7 and st.stride == 2 and net.stem_pool and st.out_channels == 64
                           and os.environ.get("LAUD_STEM_FUSED", "1") == "1")
        if self.stem_fused:
            wf = np.zeros((64, 7, 8, 4))
            wf[:, :, :7, :3] = ws.transpose(0, 2, 3, 1)  # (co, ky, kx, c)
            wf = np.concatenate([wf.reshape(64, 224), np.zeros((64, 32))], axis=1)
            self.stem_wf = torch.from_numpy(wf).to(device=device, dtype=torch.bfloat16).contiguous()
        # fused 3x3/2 stem without pool (RegNetY, laud_stem3): weights [32][ky][kx*4 + c]
        self.stem3_fused = (st.kernel == 3 and st.stride == 2 and not net.stem_pool and st.out_channels == 32
                            and os.environ.get("LAUD_STEM_FUSED", "1") == "1")
        if self.stem3_fused:
            w3 = np.zeros((32, 3, 4, 4))
            w3[:, :, :3, :3] = ws.transpose(0, 2, 3, 1)  # (co, ky, kx, c)
            self.stem_wf3 = torch.from_numpy(w3.reshape(32, 48)).to(device=device, dtype=torch.bfloat16).contiguous()
        self.stem_bias = D.fvec(params["stem_b"], st.out_channels, 0.0, device)
        self.mean = torch.tensor(IMAGENET_MEAN, dtype=torch.float32, device=device)
        self.inv_std = torch.tensor([1.0 / s for s in IMAGENET_STD], dtype=torch.float32, device=device)
        # blocks
        self.slots: list[BlockSlot] = []
        for bp in params["blocks"]:
            blk = bp["block"]
            ep = D.Epilogue(s1=bp["s1"], b1=bp["b1"], relu1=True, s2=bp["s2"], b2=bp["b2"],
                            relu2=True, s3=bp["s3"], b3=bp["b3"], sd=bp["sd"], bd=bp["bd"],
                            relu_out=True)
            db = D.DeviceBlock(blk, bp["w1"], bp["w2"], bp["w3"], bp["wd"], ep,
                               masker_w=bp["masker_w"], device=device, fold_scale=True)
            s = self.plan[bp["stage"] - 1] if para is Paradigm.SPATIAL else 0
            if para is Paradigm.CHANNEL:
                g = self.plan[bp["stage"] - 1]
                db.set_channel_masker(bp["ch_w1"], bp["ch_w2"], g)
                # grouped conv2 (RegNet): the EXT block-diagonal dense kernel
                # (laud.h w2_dense; the network executor is EXT territory anyway)
                db.enable_grouped_channel()
            if "se_w1" in bp:  # RegNetY squeeze-excitation (EXT)
                db.set_se(bp["se_w1"], bp["se_b1"], bp["se_w2"], bp["se_b2"])
            # conv1 schedule: the dilated pixel set covers most of the input for
            # S <= 2 at ratio >= 0.4 (r_dil ~0.9 at r = 0.5), where the dense
            # conv1 (contiguous TMA rows, no dilation pass) is cheaper
            db.conv1_dense = para is Paradigm.SPATIAL and (
                s <= 2 and target_ratio >= 0.4 or os.environ.get("LAUD_CONV1_DENSE_ALL", "1") == "1")
            self.slots.append(BlockSlot(bp["stage"], bp["index"], db, s))
        fc_in = net.classifier_features
        self.fc_w = D.pack_weight(params["fc_w"][:, :, None, None], D.pad8(fc_in), device)
        self.fc_b = D.fvec(params["fc_b"], net.num_classes, 0.0, device)
        self.n_cls = D.pad8(net.num_classes)
        self._bufs = {}
        self.ws = D.Workspace(device)
        # masker-conv3 fusion: block i+1 reuses block i's conv3 output dots when
        # both run on the same grid with the same S and i+1 has no downsample
        self.fuse_masker = False  # measured: the conv3 dot costs more than the masker saves
        # small grids: conv2 may split K over a thread-block cluster (laud.h
        # latency_split; a different fp32 summation order, within the logit gates)
        self.latency_split = os.environ.get("LAUD_LATENCY_SPLIT", "1") != "0"
        for i, slot in enumerate(self.slots):
            prev = self.slots[i - 1] if i > 0 else None
            b = slot.db.block
            slot.fused_in = (para is Paradigm.SPATIAL and prev is not None and prev.stage == slot.stage
                             and not b.has_downsample and b.stride == 1 and prev.s == slot.s)

    # ------------------------------------------------------------------ buffers
    def _buf(self, name, shape, dtype=torch.bfloat16):
        """View of a grow-only flat buffer (stable addresses across forwards)."""
        numel = int(np.prod(shape))
        b = self._bufs.get(name)
        if b is None or b.numel() < numel or b.dtype != dtype:
            b = torch.empty(numel, dtype=dtype, device=self.device)
            self._bufs[name] = b
        return b[:numel].view(shape)

    def _block_paradigm(self, slot: BlockSlot) -> str:
        return self.paradigm if self.paradigm in ("spatial", "layer", "channel") else "static"

    # ------------------------------------------------------------------ forward
    def forward(self, images: torch.Tensor, stream=None, record=None) -> torch.Tensor:
        """images: (N, H, W, 3) uint8 on the device -> (N, classes) fp32 logits.

        ``record`` (optional list) receives (slot, coarse, counts) references
        per dynamic block for post-hoc rate statistics.
        """
        net = self.net
        n, h, w, _ = images.shape
        k, st = self.stem_k, self.stem_stride
        pad = k // 2
        ho, wo = (h + 2 * pad - k) // st + 1, (w + 2 * pad - k) // st + 1
        sh = D.stream_handle(stream)
        if self.stem_fused and h == 224 and w == 224:
            pool = self._buf("pool", (n, 56, 56, self.stem_c))
            _lib.call("laud_stem_pool", D.ptr(images), n, h, w, D.ptr(self.mean), D.ptr(self.inv_std),
                      D.ptr(self.stem_wf), D.ptr(self.stem_bias), D.ptr(pool), sh)
            return self._blocks_and_head(pool, n, stream, record)
        if self.stem3_fused and h == 224 and w == 224:
            stem_out = self._buf("stem", (n, 112, 112, self.stem_c))
            _lib.call("laud_stem3", D.ptr(images), n, h, w, D.ptr(self.mean), D.ptr(self.inv_std),
                      D.ptr(self.stem_wf3), D.ptr(self.stem_bias), D.ptr(stem_out), sh)
            return self._blocks_and_head(stem_out, n, stream, record)
        cols = self._buf("cols", (n * ho * wo, self.stem_cols))
        _lib.call("laud_stem_im2col", D.ptr(images), n, h, w, k, st, pad, D.ptr(self.mean),
                  D.ptr(self.inv_std), D.ptr(cols), self.stem_cols, sh)
        stem_out = self._buf("stem", (n, ho, wo, self.stem_c))
        CH.conv(act=cols, in_hw=(n * ho * wo, 1), in_c=self.stem_cols, in_ld=self.stem_cols,
                weight=self.stem_w, n_out=self.stem_c, out=stem_out, out_ld=self.stem_c,
                out_hw=(ho, wo), batch=n, a_compact=1, bias=self.stem_bias,
                relu=1, stream=stream)
        x = stem_out
        if net.stem_pool:
            ph, pw = (ho - 1) // 2 + 1, (wo - 1) // 2 + 1
            pool = self._buf("pool", (n, ph, pw, self.stem_c))
            _lib.call("laud_maxpool3s2", D.ptr(stem_out), n, ho, wo, self.stem_c, D.ptr(pool), sh)
            x = pool
        return self._blocks_and_head(x, n, stream, record)

    def _aux_stream(self):
        if getattr(self, "_aux", None) is None:
            self._aux = torch.cuda.Stream(device=self.device)
        return self._aux

    def _blocks_and_head(self, x, n, stream, record):
        sh = D.stream_handle(stream)
        ping = 0
        prev_coarse = None
        for bi, slot in enumerate(self.slots):
            db = slot.db
            hh, ww = x.shape[1], x.shape[2]
            oh, ow = db.out_hw(hh, ww)
            para = self._block_paradigm(slot)
            if db.block.has_downsample:
                ping ^= 1
                out = self._buf(f"act{ping}", (n, oh, ow, db.cout_p))
            else:
                out = x  # in-place residual: conv1 reads x before conv3 writes it
            kw = {}
            if para == "spatial" and self.fuse_masker:
                # masker-conv3 fusion inside a stage: this block's conv3 accumulates
                # the next block's masker dots; the next masker reads only the
                # cells this block skipped
                ncell = n * (oh // slot.s) * (ow // slot.s)
                fused_in = slot.fused_in
                nxt = self.slots[bi + 1] if bi + 1 < len(self.slots) else None
                fused_out = nxt is not None and nxt.fused_in
                if fused_in or fused_out:
                    kw["coarse_out"] = self._buf(f"coarse{bi & 1}", (ncell,), torch.uint8)
                    kw["dn"] = self._buf("dn", (ncell,), torch.float32)
                    kw["prev_coarse"] = prev_coarse if fused_in else None
                    kw["next_wdiff"] = nxt.db.wdiff if fused_out else None
            if para in ("spatial", "layer"):
                kw["aux_stream"] = self._aux_stream()  # small grids fork the masker (laud.h aux_stream)
            if para in ("spatial", "layer", "static"):
                kw["latency_split"] = self.latency_split  # conv2 split-K: small grids / last partial wave
            y, coarse, cells, counts = db.forward(x, para, slot.s if para == "spatial" else 0,
                                                  out=out, stream=stream, ws=self.ws, **kw)
            prev_coarse = kw.get("coarse_out")
            if record is not None and para == "channel":
                record.append((slot, db._ch_coarse[: n * db.ch_d].clone(), db._ch_count[: 4 * n].clone()))
            elif record is not None and para != "static":
                ncell = n * (oh // slot.s) * (ow // slot.s) if para == "spatial" else n
                record.append((slot, coarse[:ncell].clone(), counts[:8].clone()))
            x = y
        c = x.shape[-1]
        feat = self._buf("feat", (n, c))
        _lib.call("laud_global_avgpool", D.ptr(x), n, x.shape[1] * x.shape[2], c, D.ptr(feat), sh)
        logits = self._buf("logits", (n, self.n_cls), torch.float32)
        CH.conv(act=feat, in_hw=(n, 1), in_c=c, in_ld=c, weight=self.fc_w, n_out=self.n_cls,
                out=logits, out_ld=self.n_cls, out_hw=(n, 1), batch=1, a_compact=1,
                bias=self.fc_b, out_f32=1, stream=stream)
        return logits

    # ------------------------------------------------------------------ calibration
    def calibrate(self, images: torch.Tensor, ratio: Optional[float] = None):
        """Set each dynamic block's masker bias so its active ratio ~= ``ratio``.

        Block by block on the calibration batch: run the block's masker alone,
        read the per-cell decision values d, and place the threshold at the
        (1 - ratio) quantile (bias = -quantile).  Done once, outside timing.
        """
        ratio = self.target_ratio if ratio is None else ratio
        if self.paradigm == "channel":
            return self._calibrate_channel(images, ratio)
        if self.paradigm not in ("spatial", "layer"):
            return
        for slot in self.slots:
            slot.db.masker_bias = -1e30  # placeholder; set below
        saved = []
        lib = _lib.lib()
        orig_forward = D.DeviceBlock.forward

        def hooked(db, x, paradigm="spatial", s=1, **kw):
            if paradigm in ("spatial", "layer"):
                n, h, w, cp = x.shape
                ho, wo = db.out_hw(h, w)
                ss = s if paradigm == "spatial" else ho
                cells = n * (ho // ss) * (wo // ss)
                npart = lib.laud_masker_partial_floats(n, h, w, cp, ss, db.block.stride)
                part = torch.empty(max(1, npart), dtype=torch.float32, device=x.device)
                coarse = torch.empty(cells, dtype=torch.uint8, device=x.device)
                lst = torch.empty(cells, dtype=torch.int32, device=x.device)
                cnt = torch.zeros(1, dtype=torch.int32, device=x.device)
                scan = self.ws.get("scan", lib.laud_scan_workspace_bytes(max(cells, n * h * w)), zero=True)
                _lib.call("laud_spatial_masker", D.ptr(x), 0, cp, n, h, w, cp, ss, db.block.stride,
                          D.ptr(db.wdiff), 0.0, D.ptr(coarse), D.ptr(lst), D.ptr(cnt), D.ptr(part),
                          D.ptr(scan), D.stream_handle())
                win = ss * db.block.stride
                dbar = part.view(cells, -1).sum(1) / float(win * win)
                q = torch.quantile(dbar.double(), 1.0 - ratio).item()
                db.masker_bias = float(-q)
                saved.append(db.masker_bias)
            return orig_forward(db, x, paradigm, s, **kw)

        D.DeviceBlock.forward = hooked
        try:
            self.forward(images)
        finally:
            D.DeviceBlock.forward = orig_forward
        torch.cuda.synchronize()
        return saved

    def _calibrate_channel(self, images: torch.Tensor, ratio: float):
        """Channel paradigm: per block, the bias on the masker's logit gaps that
        keeps ``ratio`` of the D channel groups on the calibration batch."""
        saved = []
        orig_forward = D.DeviceBlock.forward

        def hooked(db, x, paradigm="spatial", s=1, **kw):
            if paradigm == "channel":
                n, h, w, cp = x.shape
                d, cmp = db.ch_d, db.cmid_p
                dv = torch.empty(n * d, dtype=torch.float32, device=x.device)
                tmp8 = torch.empty(n * max(d, cmp), dtype=torch.uint8, device=x.device)
                exp = torch.empty(n * cmp, dtype=torch.uint8, device=x.device)
                sel = torch.empty(n * cmp, dtype=torch.int32, device=x.device)
                cnt = torch.empty(n, dtype=torch.int32, device=x.device)
                _lib.call("laud_channel_masker", D.ptr(x), 0, cp, n, h * w, cp, D.ptr(db.ch_w1),
                          db.ch_hidden, D.ptr(db.ch_w2), d, db.ch_g, d * db.ch_g, cmp, D.ptr(tmp8),
                          D.ptr(dv), D.ptr(exp), D.ptr(sel), D.ptr(cnt), None, D.stream_handle())
                q = torch.quantile(dv.double(), 1.0 - ratio).item()
                db.set_channel_bias(-q)
                saved.append(-q)
            return orig_forward(db, x, paradigm, s, **kw)

        D.DeviceBlock.forward = hooked
        try:
            self.forward(images)
        finally:
            D.DeviceBlock.forward = orig_forward
        torch.cuda.synchronize()
        return saved

    def masker_biases(self):
        if self.paradigm == "channel":
            return [getattr(slot.db, "ch_bias_value", 0.0) for slot in self.slots]
        return [slot.db.masker_bias for slot in self.slots]

    def set_masker_biases(self, biases):
        for slot, b in zip(self.slots, biases):
            if self.paradigm == "channel":
                slot.db.set_channel_bias(float(b))
            else:
                slot.db.masker_bias = float(b)

    def rate_stats(self, images: torch.Tensor):
        """Per-block measured activation ratio (host sync; not for timing)."""
        rec = []
        self.forward(images, record=rec)
        torch.cuda.synchronize()
        out = []
        for slot, coarse, counts in rec:
            if self.paradigm == "channel":
                out.append(dict(stage=slot.stage, index=slot.index, g=slot.db.ch_g,
                                r=float(coarse.float().mean().item()),
                                kept=int(counts.view(torch.int32).sum().item())))
                continue
            out.append(dict(stage=slot.stage, index=slot.index, s=slot.s,
                            r=float(coarse.float().mean().item()),
                            patches=int(counts.view(torch.int32)[0].item())))
        return out


class PipelinedRunner:
    """Streams host image batches through a LaudNetwork end to end.

    Two device input buffers, one captured CUDA graph per buffer: the pinned
    host->device upload of batch i+1 runs on a copy stream while batch i's
    forward runs; each batch's fp32 logits come back to pinned host memory on
    the compute stream right after its graph.  ``run`` returns the device-timed
    milliseconds of the whole sequence (CUDA events on the compute stream).
    """

    def __init__(self, net: "LaudNetwork", batch: int, h: int = 224, w: int = 224, warmup: int = 2):
        self.net = net
        self.bufs = [torch.empty((batch, h, w, 3), dtype=torch.uint8, device=net.device) for _ in range(2)]
        self.copy = torch.cuda.Stream(device=net.device)
        self.comp = torch.cuda.Stream(device=net.device)
        self.graphs = []
        self.logits = None
        for buf in self.bufs:
            with torch.cuda.stream(self.comp):
                for _ in range(max(1, warmup)):
                    net.forward(buf)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self.comp):
                self.logits = net.forward(buf)
            self.graphs.append(g)
        torch.cuda.synchronize()

    def run(self, host_batches, host_out, before_step=None) -> float:
        """host_batches: pinned uint8 (N, H, W, 3) tensors; host_out: pinned fp32
        (len, N, classes) tensor receiving the logits."""
        up = [torch.cuda.Event() for _ in range(2)]
        done = [torch.cuda.Event() for _ in range(2)]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        self.copy.wait_stream(torch.cuda.current_stream())
        self.comp.wait_stream(torch.cuda.current_stream())
        e0.record(self.comp)
        self.copy.wait_event(e0)
        for i, hb in enumerate(host_batches):
            k = i & 1
            with torch.cuda.stream(self.copy):
                if i >= 2:
                    self.copy.wait_event(done[k])  # graph i-2 finished reading this buffer
                self.bufs[k].copy_(hb, non_blocking=True)
                up[k].record(self.copy)
            with torch.cuda.stream(self.comp):
                if before_step is not None:
                    before_step()
                self.comp.wait_event(up[k])
                self.graphs[k].replay()
                done[k].record(self.comp)
                host_out[i].copy_(self.logits, non_blocking=True)
        e1.record(self.comp)
        e1.synchronize()
        return e0.elapsed_time(e1)


def add_channel_maskers(params: dict, gplan, seed: int = 0) -> dict:
    """Channel-masker MLP weights per block (`reference.py:189-223`): G from the
    stage's plan entry, D = C_mid / G, hidden h = max(D // 16, 16); w1 [h, C_in]
    ~ N(0, 1/C_in), w2 [2D, h] ~ N(0, 1/h).  Stored in ``params["blocks"]`` so the
    oracle composer runs the same maskers."""
    rng = np.random.default_rng(seed + 7919)
    for bp in params["blocks"]:
        blk = bp["block"]
        g = int(gplan[bp["stage"] - 1])
        d = blk.conv2.out_channels // g
        h = max(d // 16, 16)
        ci = blk.input_shape.channels
        bp["ch_g"] = g
        bp["ch_w1"] = rng.standard_normal((h, ci)) / np.sqrt(ci)
        bp["ch_w2"] = rng.standard_normal((2 * d, h)) / np.sqrt(h)
    return params


def random_images(n: int, h: int = 224, w: int = 224, seed: int = 0, device="cuda") -> torch.Tensor:
    g = torch.Generator(device="cpu").manual_seed(seed)
    return torch.randint(0, 256, (n, h, w, 3), dtype=torch.uint8, generator=g).to(device)

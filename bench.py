"""Benchmark: LAUDNet-ResNet-101 (spatial S=4-2-2-1, ratio 0.5) images/s on B200.

Contract (one JSON line on rank 0):
  python bench.py --gpus N --steps K --warmup W [--impl reference]
For N>1 run under torchrun: one process per GPU, weak scaling (each rank
processes its own batch of --batch images), no collective on the data path;
the timed region is bracketed by barriers and the max over ranks is reported.

Step = one forward of the whole LAUD-R101 (stem, 33 dynamic bottleneck
blocks with their maskers computed inside the step, GAP, FC) over a batch of
synthetic 224x224 uint8 images already resident in HBM, replayed as one CUDA
graph.  L2 is flushed (256 MiB write) before every timed step and each step
is timed with CUDA events on the launching stream.  ``e2e`` repeats the step
through the public API with the pinned-host image upload and the logits
download inside the timed region.  ``--impl reference`` times the CPU
oracle (numpy fp64 restatement of the reference executor) on this host.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="laud", choices=["laud", "reference"])
    ap.add_argument("--arch", default="resnet101")
    ap.add_argument("--paradigm", default="spatial", choices=["spatial", "channel", "layer", "static"])
    ap.add_argument("--plan", default=None, help="S per stage (spatial, default 4-2-2-1) or "
                    "G per stage (channel, default 1-1-1-1)")
    ap.add_argument("--ratio", type=float, default=0.5)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--no-baselines", action="store_true", help="skip static / cuDNN / CPU / sweep legs")
    ap.add_argument("--cpu-images", type=int, default=24)  # ~10 s of host CPU work
    a = ap.parse_args()
    if a.plan is None:
        a.plan = "1-1-1-1" if a.paradigm == "channel" else "4-2-2-1"
    return a


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# reference arm: CPU oracle
# ---------------------------------------------------------------------------


def cpu_oracle_images_per_s(args, n_images, params=None, biases=None):
    from oracle import laud_oracle as O
    from paper_2308_15949_b200.network import make_params
    params = params or make_params(args.arch, 0)
    plan = tuple(int(v) for v in args.plan.split("-"))
    rng = np.random.default_rng(1)
    img = rng.integers(0, 256, (1, 224, 224, 3), dtype=np.uint8)
    t = []
    for _ in range(n_images):
        t0 = time.perf_counter()
        O.network_forward(params, img, args.paradigm, plan, biases)
        t.append(time.perf_counter() - t0)
    return 1.0 / statistics.median(t), t


def blas_threads():
    try:
        import threadpoolctl
        info = threadpoolctl.threadpool_info()
        n = sum(i.get("num_threads", 0) for i in info if i.get("user_api") == "blas")
        return n or os.cpu_count()
    except Exception:
        return os.cpu_count()


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from paper_2308_15949_b200.network import add_channel_maskers, make_params
    params = make_params(args.arch, 0)
    plan = tuple(int(v) for v in args.plan.split("-"))
    if args.paradigm == "channel":
        add_channel_maskers(params, plan, 0)
    from oracle import laud_oracle as O
    img = np.random.default_rng(1).integers(0, 256, (1, 224, 224, 3), dtype=np.uint8)
    for _ in range(max(1, min(args.warmup, 1))):
        O.network_forward(params, img, args.paradigm, plan)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.network_forward(params, img, args.paradigm, plan)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    v = args.steps / tot
    cores = blas_threads()
    line = {
        "impl": "reference", "metric": "images_per_sec", "value": v, "unit": "images/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"LAUD-{args.arch} {args.paradigm} S={args.plan} r={args.ratio}, "
                               "1 image per step (bounded CPU sample)",
                   "arch": args.arch, "plan": args.plan, "ratio": args.ratio},
        "cpu_baseline": {"value": v, "unit": "images/s", "cores": cores, "kind": "port",
                         "sample": "1 synthetic 224x224 image per step through the numpy fp64 "
                                   "oracle network (oracle/laud_oracle.py)"},
        "e2e": {"value": v, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []  # (host time, csv line)
        self.window = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def wait_ready(self, timeout=10.0):
        """Block until nvidia-smi streams samples (it takes ~0.1-1 s to start)."""
        t0 = time.time()
        while self.proc and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.02)

    def mark(self, t0, t1):
        """Keep only the samples taken inside [t0, t1] (the timed region)."""
        self.window = (t0, t1)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = [ln for ts, ln in self.lines
                 if self.window is None or self.window[0] <= ts <= self.window[1] + 0.03]
        for ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = max(smax, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------


def timed_graph(torch, graph, steps, flush, stream):
    """Sum of per-step event times, L2 flushed before each step (outside events)."""
    tot = 0.0
    per = []
    for _ in range(steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        graph.replay()
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        per.append(ms)
        tot += ms
    return tot, per


def capture(torch, fn, warmup):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(max(1, warmup)):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out = fn()
    torch.cuda.synchronize()
    return g, out


def _alg(r):
    """Algorithmic FLOPs and compulsory bytes of one conv-engine launch."""
    flops = 2.0 * r.rows * r.n_out * r.k
    cin = r.k // max(1, r.taps)
    nbytes = 2.0 * r.rows * (cin + r.n_out * (2 if r.resid else 1))
    return flops, nbytes


def conv_roofline(torch, net, images, pk, pk_kind):
    """Per-launch CUDA-event profile of one eager forward (outside the timed region).

    The roofline object describes the dominant launch shape of the conv engine
    (largest total time in the step): achieved = algorithmic FLOPs (or bytes,
    whichever bounds it) per launch / average launch duration of that shape.
    """
    from paper_2308_15949_b200 import _lib
    lib = _lib.lib()
    torch.cuda.synchronize()
    lib.laud_profile_begin()
    net.forward(images)
    recs = (_lib.ProfileRecord * 4096)()
    n = lib.laud_profile_end(recs, 4096)
    recs = recs[:n]
    convs = [r for r in recs if r.tag == 0]
    maskers = [r for r in recs if r.tag == 1]
    all_ms = sum(r.ms for r in recs)
    groups = {}
    for r in convs:
        key = (r.rows, r.n_out, r.k, r.taps, r.resid)
        groups.setdefault(key, []).append(r)
    key, grp = max(groups.items(), key=lambda kv: sum(x.ms for x in kv[1]))
    flops, nbytes = _alg(grp[0])
    avg_ms = sum(x.ms for x in grp) / len(grp)
    peak_t = pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
    peak_b = pk["hbm_gbs"]
    t_tensor = flops / (peak_t * 1e12)
    t_hbm = nbytes / (peak_b * 1e9)
    if t_tensor >= t_hbm:
        bound, ach, peak, unit = "tensor", flops / (avg_ms * 1e-3) / 1e12, peak_t, "TFLOP/s"
    else:
        bound, ach, peak, unit = "hbm", nbytes / (avg_ms * 1e-3) / 1e9, peak_b, "GB/s"
    tot_f = sum(_alg(r)[0] for r in convs)
    tot_ms = sum(r.ms for r in convs)
    # step-level roofline of the conv engine: slower of FLOPs and bytes per launch, summed
    ideal_ms = sum(max(_alg(r)[0] / (peak_t * 1e12), _alg(r)[1] / (peak_b * 1e9)) for r in convs) * 1e3
    mb = sum(r.bytes for r in maskers)
    mms = sum(r.ms for r in maskers)
    rows, n_out, k, taps, resid = key
    return {
        "kernel": f"laud::conv_gemm_kernel, dominant shape rows={rows} n_out={n_out} K={k} "
                  f"taps={taps} resid={resid} ({len(grp)} launches/step)",
        "shape": f"rows={rows} n_out={n_out} K={k} taps={taps} resid={resid}",
        "bound": bound, "achieved": round(ach, 2), "peak": peak, "unit": unit,
        "frac": round(ach / peak, 4), "traffic": None,
        "peak_source": f"{pk_kind} MEASURED_PEAKS.json ({'bf16_tflops_sustained' if bound == 'tensor' else 'hbm_gbs'})",
        "alg_flops_per_launch": flops, "alg_bytes_per_launch": nbytes,
        "avg_launch_us": round(avg_ms * 1e3, 2),
        "share_of_profiled_step": round(sum(x.ms for x in grp) / all_ms, 3) if all_ms else None,
        "engine_all_launches": {"launches": len(convs), "ms": round(tot_ms, 3),
                                "tflops": round(tot_f / (tot_ms * 1e-3) / 1e12, 1),
                                "roofline_ms": round(ideal_ms, 3),
                                "frac_of_roofline": round(ideal_ms / tot_ms, 4),
                                "share_of_step": round(tot_ms / all_ms, 3) if all_ms else None},
        "masker_gbs": round(mb / (mms * 1e-3) / 1e9, 1) if mms else None,
    }


TV_MODELS = {"resnet50": "resnet50", "resnet101": "resnet101", "regnety-400mf": "regnet_y_400mf",
             "regnety-800mf": "regnet_y_800mf", "regnety-1.6gf": "regnet_y_1_6gf"}


def static_cudnn_ms(torch, batch, steps, warmup, flush, arch="resnet101"):
    """torchvision static model of the same arch (RegNetY includes its SE blocks),
    channels_last bf16, CUDA graph: the library (cuDNN) static baseline."""
    try:
        import torchvision
    except Exception:
        return None
    m = getattr(torchvision.models, TV_MODELS[arch])().cuda().eval().to(memory_format=torch.channels_last).bfloat16()
    x = torch.randn(batch, 3, 224, 224, device="cuda").bfloat16().to(memory_format=torch.channels_last)
    with torch.no_grad():
        g, _ = capture(torch, lambda: m(x), warmup)
        tot, _ = timed_graph(torch, g, steps, flush, torch.cuda.current_stream())
    del m, g
    torch.cuda.empty_cache()
    return tot / steps


def batch1_latency(torch, args, net, flush, reps=20):
    """BASELINE config 3's latency leg: one image, whole network as one CUDA graph
    (L2 flushed before each replay): the dynamic net (its calibrated maskers),
    the in-house static net and the torchvision/cuDNN static net, median ms."""
    from paper_2308_15949_b200.network import LaudNetwork, random_images
    img = random_images(1, seed=7)

    def med(g):
        _, per = timed_graph(torch, g, reps, flush, torch.cuda.current_stream())
        return round(float(np.median(per)), 4)

    out = {}
    g, _ = capture(torch, lambda: net.forward(img), 2)
    out["laud"] = med(g)
    del g
    snet = LaudNetwork(args.arch, "static", args.plan, 1.0, seed=0)
    g, _ = capture(torch, lambda: snet.forward(img), 2)
    out["static_inhouse"] = med(g)
    del g, snet
    try:
        import torchvision
        m = getattr(torchvision.models, TV_MODELS[args.arch])().cuda().eval().to(
            memory_format=torch.channels_last).bfloat16()
        x = torch.randn(1, 3, 224, 224, device="cuda").bfloat16().to(memory_format=torch.channels_last)
        with torch.no_grad():
            g, _ = capture(torch, lambda: m(x), 2)
            out["static_cudnn"] = med(g)
        del g, m
    except Exception:
        out["static_cudnn"] = None
    torch.cuda.empty_cache()
    return out


def block_sweep_b1_vs_cpu(torch, args, flush, reps_cpu=3):
    """Per-block latency vs activation ratio at batch 1 (SURVEY §8d CPU baseline):
    the device (CUDA graph, L2 flushed) next to the numpy fp64 oracle's
    ``block_forward_sparse`` (the reference's algorithm) on this box's host
    cores, same block geometry, exact-count masks, median of ``reps_cpu``."""
    from oracle import laud_oracle as O
    from paper_2308_15949_b200 import device as D
    from paper_2308_15949_b200.core import DynamicConfig, Paradigm
    from paper_2308_15949_b200.network import make_params
    params = make_params(args.arch, 0)
    plan = tuple(int(v) for v in args.plan.split("-"))
    out = {}
    rng = np.random.default_rng(0)
    seen = set()
    for bp in params["blocks"]:
        if bp["stage"] in seen or bp["index"] != 1:
            continue
        seen.add(bp["stage"])
        blk = bp["block"]
        s = plan[bp["stage"] - 1]
        db = D.DeviceBlock(blk, bp["w1"], bp["w2"], bp["w3"], None)
        wsp = D.Workspace()
        ci, o = blk.input_shape, blk.output_shape
        xh = rng.standard_normal((1, ci.channels, ci.height, ci.width))
        x = D.to_device_nhwc(xh)
        cells = (o.height // s) * (o.width // s)
        bw = O.BlockWeights(bp["w1"], bp["w2"], bp["w3"], None)
        row = {}
        for r in (0.2, 0.5, 0.8, 1.0, "static"):
            if r == "static":
                fn = lambda: db.forward(xx, "static", out=xx, ws=wsp)  # noqa: E731
                cfg, om = DynamicConfig(Paradigm.STATIC), None
            else:
                cz = np.zeros(cells, np.uint8)
                cz[rng.permutation(cells)[:int(round(r * cells))]] = 1
                coarse = torch.from_numpy(cz).cuda()
                fn = lambda: db.forward(xx, "spatial", s, coarse=coarse, out=xx, ws=wsp)  # noqa: E731
                c3 = cz.reshape(1, o.height // s, o.width // s).astype(bool)
                cfg = DynamicConfig(Paradigm.SPATIAL, spatial_granularity=s)
                om = O.SpatialMask(c3, O.upsample_coarse(c3, s), s)
            xx = x.clone()
            g, _ = capture(torch, fn, 2)
            tot, _ = timed_graph(torch, g, 20, flush, torch.cuda.current_stream())
            del g
            ts = []
            for _ in range(reps_cpu):
                t0 = time.perf_counter()
                O.block_forward_sparse(xh, bw, blk, cfg, om)
                ts.append(time.perf_counter() - t0)
            row[str(r)] = {"gpu_us": round(1e3 * tot / 20, 1),
                           "cpu_oracle_us": round(1e6 * statistics.median(ts), 1)}
        out[f"s{bp['stage']}b1_S{s}"] = row
    return {"blocks": out, "cpu_cores": blas_threads(), "cpu_kind": "port (numpy fp64 oracle)",
            "batch": 1}


def block_sweep(torch, args, flush):
    """Per-block device latency vs activation ratio (exact-count masks), batch = args.batch."""
    from paper_2308_15949_b200 import device as D
    from paper_2308_15949_b200.network import make_params
    params = make_params(args.arch, 0)
    plan = tuple(int(v) for v in args.plan.split("-"))
    out = {}
    rng = np.random.default_rng(0)
    seen = set()
    for bp in params["blocks"]:
        if bp["stage"] in seen or bp["index"] != 1:
            continue
        seen.add(bp["stage"])
        blk = bp["block"]
        s = plan[bp["stage"] - 1]
        ep = D.Epilogue(s1=bp["s1"], b1=bp["b1"], relu1=True, s2=bp["s2"], b2=bp["b2"], relu2=True,
                        s3=bp["s3"], b3=bp["b3"], relu_out=True)
        db = D.DeviceBlock(blk, bp["w1"], bp["w2"], bp["w3"], None, ep, fold_scale=True)
        wsp = D.Workspace()
        n = args.batch
        h = blk.input_shape.height
        x = torch.randn(n, h, h, db.cin_p, device="cuda").relu_().bfloat16()
        o = blk.output_shape
        cells = (o.height // s) * (o.width // s)
        row = {}
        for r in (0.2, 0.5, 0.8, 1.0):
            xx = x.clone()
            if args.paradigm == "channel":
                # exact-count per-sample channel masks (G = plan entry), SURVEY §8(d) config 4
                cm, g_ = blk.conv2.out_channels, s
                d = cm // g_
                k = int(round(r * d))
                mm = np.zeros((n, db.cmid_p), np.uint8)
                for i in range(n):
                    keep = np.repeat(np.isin(np.arange(d), rng.permutation(d)[:k]), g_)
                    mm[i, :cm] = keep
                chm = torch.from_numpy(mm.reshape(-1)).cuda()
                fn = lambda: db.forward(xx, "channel", out=xx, ws=wsp, chmask=chm)  # noqa: E731
            else:
                k = int(round(r * cells))
                cz = np.zeros((n, cells), np.uint8)
                for i in range(n):
                    cz[i, rng.permutation(cells)[:k]] = 1
                coarse = torch.from_numpy(cz.reshape(-1)).cuda()
                fn = lambda: db.forward(xx, "spatial", s, coarse=coarse, out=xx, ws=wsp)  # noqa: E731
            g, _ = capture(torch, fn, 2)
            tot, _ = timed_graph(torch, g, 10, flush, torch.cuda.current_stream())
            row[str(r)] = round(1e3 * tot / 10, 1)
            del g
        xx = x.clone()
        g, _ = capture(torch, lambda: db.forward(xx, "static", out=xx, ws=wsp), 2)
        tot, _ = timed_graph(torch, g, 10, flush, torch.cuda.current_stream())
        row["static"] = round(1e3 * tot / 10, 1)
        out[f"s{bp['stage']}b1_{'G' if args.paradigm == 'channel' else 'S'}{s}"] = row
    return out


def run_gpu(args):
    import torch
    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    else:
        torch.cuda.set_device(0)
    from paper_2308_15949_b200 import _lib
    from paper_2308_15949_b200.network import LaudNetwork, random_images
    pk, pk_kind = peaks()
    lib = _lib.lib()

    net = LaudNetwork(args.arch, args.paradigm, args.plan, args.ratio, seed=0)
    images = random_images(args.batch, seed=1000 + rank)
    net.calibrate(images)
    rates = net.rate_stats(images) if args.paradigm != "static" else []
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    # launches of our kernels per step (host-side count of one eager forward)
    c0 = lib.laud_launch_count()
    net.forward(images)
    torch.cuda.synchronize()
    launches_per_step = lib.laud_launch_count() - c0

    graph, logits = capture(torch, lambda: net.forward(images), args.warmup)
    for _ in range(args.warmup):
        flush.zero_()
        graph.replay()
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        clk.wait_ready()
        t_start = time.time()
        tot_ms, per = timed_graph(torch, graph, args.steps, flush, stream)
        clk.mark(t_start, time.time())
    torch.cuda.synchronize()
    if ws > 1:
        t = torch.tensor([tot_ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        tot_ms = float(t.item())
        torch.distributed.barrier()
    ms_step = tot_ms / args.steps
    value = ws * args.batch * args.steps / (tot_ms * 1e-3)

    # ---- e2e: pinned host images -> device, forward, logits -> host, every step,
    # through the public streaming runner (upload of batch i+1 overlaps batch i)
    from paper_2308_15949_b200.network import PipelinedRunner
    host_img = torch.empty(images.shape, dtype=torch.uint8, pin_memory=True)
    host_img.copy_(images.cpu())
    n_cls = logits.shape[1]
    host_out = torch.empty((args.steps, args.batch, n_cls), dtype=torch.float32, pin_memory=True)
    runner = PipelinedRunner(net, args.batch, images.shape[1], images.shape[2])
    runner.run([host_img] * 2, host_out)  # warm
    if ws > 1:
        torch.distributed.barrier()
    e_tot = runner.run([host_img] * args.steps, host_out, before_step=flush.zero_)
    if ws > 1:
        t = torch.tensor([e_tot], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e_tot = float(t.item())
    e2e = {"value": ws * args.batch * args.steps / (e_tot * 1e-3), "unit": "images/s",
           "h2d_bytes_per_step": int(host_img.numel()), "d2h_bytes_per_step": int(args.batch * n_cls * 4),
           "path": "network.PipelinedRunner (public API): per step a pinned uint8 upload (copy stream, "
                   "overlapping the previous step's forward), the forward as a CUDA graph and the fp32 "
                   "logits download; the 256 MiB L2 flush before every step is inside the timed region"}
    del runner

    extra = {}
    roof = conv_roofline(torch, net, images, pk, pk_kind)
    prof = ROOT / "profiles" / "conv_traffic.json"
    if prof.exists():  # ncu --set full dram bytes of the same launch shape (profiles/)
        try:
            t = json.loads(prof.read_text())
            if t.get("shape") == roof.get("shape"):
                roof["traffic"] = t.get("traffic_per_launch")
        except Exception:
            pass
    if rank == 0 and not args.no_baselines and ws == 1:
        # static baselines on the same weights and a cuDNN library baseline
        snet = LaudNetwork(args.arch, "static", args.plan, 1.0, seed=0)
        sg, _ = capture(torch, lambda: snet.forward(images), 2)
        s_tot, _ = timed_graph(torch, sg, max(3, args.steps // 2), flush, stream)
        static_ms = s_tot / max(3, args.steps // 2)
        del sg, snet
        torch.cuda.empty_cache()
        cud = static_cudnn_ms(torch, args.batch, max(3, args.steps // 2), 2, flush, args.arch)
        extra["static_inhouse_ms"] = round(static_ms, 3)
        extra["static_cudnn_ms"] = round(cud, 3) if cud else None
        extra["latency_reduction_vs_static_inhouse"] = round(1 - ms_step / static_ms, 4)
        if cud:
            extra["latency_reduction_vs_static_cudnn"] = round(1 - ms_step / cud, 4)
        try:
            extra["batch1_latency_ms"] = batch1_latency(torch, args, net, flush)
        except Exception as exc:
            extra["batch1_latency_ms"] = f"failed: {exc!r}"
        try:
            extra["per_block_us_vs_ratio"] = block_sweep(torch, args, flush)
        except Exception as exc:  # never lose the headline line to the sweep
            extra["per_block_us_vs_ratio"] = f"failed: {exc!r}"
        if args.paradigm == "spatial" and ws == 1:
            try:
                extra["per_block_b1_vs_cpu"] = block_sweep_b1_vs_cpu(torch, args, flush)
            except Exception as exc:
                extra["per_block_b1_vs_cpu"] = f"failed: {exc!r}"
    cpu = None
    if rank == 0 and ws == 1 and not args.no_baselines:
        v, ts = cpu_oracle_images_per_s(args, args.cpu_images, params=net.params,
                                        biases=net.masker_biases())
        cpu = {"value": round(v, 4), "unit": "images/s", "cores": blas_threads(), "kind": "port",
               "sample": f"{args.cpu_images} synthetic images, batch 1, through the numpy fp64 oracle "
                         f"network (same weights and masker biases), median of {len(ts)}"}
    if rank == 0:
        r_mean = float(np.mean([r["r"] for r in rates])) if rates else 1.0
        line = {
            "metric": "images_per_sec", "value": round(value, 2), "unit": "images/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic",
            "config": {"workload": f"LAUDNet-{args.arch} {args.paradigm} S={args.plan} ratio {args.ratio}, "
                                   f"224x224, batch {args.batch} per GPU (BASELINE config 3, throughput)",
                       "global_batch": ws * args.batch, "arch": args.arch, "plan": args.plan,
                       "target_ratio": args.ratio, "measured_ratio_mean": round(r_mean, 4),
                       "l2_policy": "256 MiB L2 flush before every timed step",
                       "parallelism": f"batch-shard x{ws} (no collective on the hot path)",
                       "graph": True},
            "e2e": e2e, "roofline": roof, "cpu_baseline": cpu, "gpu_launches": int(launches_per_step * args.steps),
            "clocks": clk.summary(),
        }
        line.update(extra)
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()

"""Network shape source: bottleneck block lists and per-stage S/G plans.

Mirrors the spec-building half of ``dynlat.zoo``: ``.net`` text format
(`pkg/src/dynlat/zoo.py:130-157`), block assembly `_build` (`zoo.py:160-216`:
mid = width // bottleneck, groups = mid // group_width, stride on the first
block of a stage, downsample iff stride > 1 or width change, chaining check),
``build_network`` (`zoo.py:219-241`), ``parse_plan`` (`zoo.py:244-270`) and
``config_for_stage`` (`zoo.py:281-291`).  The latency/sweep half of zoo.py is
the analytical predictor and is out of scope.

Architectures are kept as in-code tables (same six stage fields as the
reference's ``.net`` rows); ``regnety-1.6gf`` is added for BASELINE config 5
(torchvision RegNetY-1.6GF: depths 2-6-17-2, widths 48-120-336-888, group
width 24, SE 1/4, 3x3/s2 stem with 32 channels and no pool).
"""

from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path
from typing import Optional, Union

from .core import BlockSpec, ConvLayerSpec, DynamicConfig, Paradigm, TensorShape
from .errors import (GranularityMismatch, PlanLengthMismatch, SpecFileError,
                     UnknownNetwork)

# name -> (header fields, stage rows (depth, width, bottleneck, group_width, se, stride))
_ARCH = {
    "resnet50": (
        dict(input=(224, 224), stem_width=64, stem_kernel=7, stem_stride=2,
             stem_pool=True, classes=1000),
        [(3, 256, 4, 0, 0, 1), (4, 512, 4, 0, 0, 2), (6, 1024, 4, 0, 0, 2),
         (3, 2048, 4, 0, 0, 2)]),
    "resnet101": (
        dict(input=(224, 224), stem_width=64, stem_kernel=7, stem_stride=2,
             stem_pool=True, classes=1000),
        [(3, 256, 4, 0, 0, 1), (4, 512, 4, 0, 0, 2), (23, 1024, 4, 0, 0, 2),
         (3, 2048, 4, 0, 0, 2)]),
    "regnety-400mf": (
        dict(input=(224, 224), stem_width=32, stem_kernel=3, stem_stride=2,
             stem_pool=False, classes=1000),
        [(1, 48, 1, 8, 4, 2), (3, 104, 1, 8, 4, 2), (6, 208, 1, 8, 4, 2),
         (6, 440, 1, 8, 4, 2)]),
    "regnety-800mf": (
        dict(input=(224, 224), stem_width=32, stem_kernel=3, stem_stride=2,
             stem_pool=False, classes=1000),
        [(1, 64, 1, 16, 4, 2), (3, 128, 1, 16, 4, 2), (8, 320, 1, 16, 4, 2),
         (2, 768, 1, 16, 4, 2)]),
    "regnety-1.6gf": (
        dict(input=(224, 224), stem_width=32, stem_kernel=3, stem_stride=2,
             stem_pool=False, classes=1000),
        [(2, 48, 1, 24, 4, 2), (6, 120, 1, 24, 4, 2), (17, 336, 1, 24, 4, 2),
         (2, 888, 1, 24, 4, 2)]),
}


@dataclass(frozen=True)
class BlockInstance:
    stage: int
    index: int
    block: BlockSpec


@dataclass(frozen=True)
class StageSpec:
    depth: int
    block_template: BlockSpec
    stride_first: bool


@dataclass(frozen=True)
class NetworkSpec:
    name: str
    stem: ConvLayerSpec
    stem_pool: bool
    stages: tuple
    blocks: tuple
    classifier_features: int
    num_classes: int
    input_shape: TensorShape

    def stage_feature(self, stage: int) -> TensorShape:
        return self.stages[stage - 1].block_template.output_shape

    def template_block(self, stage: int) -> BlockSpec:
        return self.stages[stage - 1].block_template

    def stem_output(self) -> TensorShape:
        h, w = self.stem.out_hw(self.input_shape.height, self.input_shape.width)
        if self.stem_pool:
            h, w = (h - 1) // 2 + 1, (w - 1) // 2 + 1
        return TensorShape(self.stem.out_channels, h, w)


@dataclass(frozen=True)
class GranularityPlan:
    paradigm: Paradigm
    values: tuple

    @property
    def text(self) -> str:
        return "-".join(map(str, self.values))


def network_preset_names() -> tuple:
    return tuple(sorted(_ARCH))


def parse_net_text(text: str, path: str = "<net>"):
    """Parse the reference's ``.net`` key=value format (`zoo.py:130-157`)."""
    header, rows = {}, []
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise SpecFileError(f"{path}:{lineno}: expected 'key = value'")
        key, val = (p.strip() for p in line.split("=", 1))
        if key == "stage":
            parts = val.split()
            if len(parts) != 6:
                raise SpecFileError(f"{path}:{lineno}: stage needs 6 fields "
                                    "(depth width bottleneck group_width se_reduction stride)")
            rows.append(tuple(int(p) for p in parts))
        else:
            header[key] = val
    need = ("name", "input", "stem_width", "stem_kernel", "stem_stride", "stem_pool", "classes")
    missing = [k for k in need if k not in header]
    if missing:
        raise SpecFileError(f"{path}: missing keys {missing}")
    if not rows:
        raise SpecFileError(f"{path}: no stages")
    h, w = (int(v) for v in header["input"].split("x"))
    fields = dict(name=header["name"], input=(h, w), stem_width=int(header["stem_width"]),
                  stem_kernel=int(header["stem_kernel"]), stem_stride=int(header["stem_stride"]),
                  stem_pool=header["stem_pool"].lower() in ("yes", "true", "1"),
                  classes=int(header["classes"]))
    return fields, rows


def _assemble(name, fields, rows, path, input_hw=None) -> NetworkSpec:
    h, w = input_hw if input_hw is not None else fields["input"]
    stem = ConvLayerSpec(3, fields["stem_width"], fields["stem_kernel"], fields["stem_stride"])
    fh, fw = stem.out_hw(h, w)
    if fields["stem_pool"]:
        fh, fw = (fh - 1) // 2 + 1, (fw - 1) // 2 + 1
    prev_c, prev_out = stem.out_channels, None
    blocks, stages = [], []
    for si, (depth, width, bneck, gw, se, stride) in enumerate(rows, start=1):
        mid = width // bneck
        groups = mid // gw if gw else 1
        stage_blocks = []
        for b in range(depth):
            s = stride if b == 0 else 1
            cin = prev_c if b == 0 else width
            blk = BlockSpec(
                conv1=ConvLayerSpec(cin, mid, 1),
                conv2=ConvLayerSpec(mid, mid, 3, s, groups),
                conv3=ConvLayerSpec(mid, width, 1),
                input_shape=TensorShape(cin, fh, fw),
                se_reduction=se or None,
                has_downsample=(b == 0 and (s > 1 or cin != width)),
            )
            if prev_out is not None and blk.input_shape != prev_out:
                raise SpecFileError(f"{path}: block chaining broken entering stage {si}")
            prev_out = blk.output_shape
            fh, fw = prev_out.height, prev_out.width
            stage_blocks.append(BlockInstance(si, b, blk))
        tmpl = stage_blocks[1].block if depth > 1 else stage_blocks[0].block
        stages.append(StageSpec(depth, tmpl, stride > 1))
        blocks.extend(stage_blocks)
        prev_c = width
    return NetworkSpec(name, stem, fields["stem_pool"], tuple(stages), tuple(blocks),
                       prev_c, fields["classes"], TensorShape(3, h, w))


def build_network(source: Union[str, Path],
                  input_hw: Optional[tuple] = None) -> NetworkSpec:
    """Preset name or ``.net`` path -> NetworkSpec (`zoo.py:219-241`)."""
    s = str(source)
    if isinstance(source, Path) or s.endswith(".net") or "/" in s:
        p = Path(source)
        if not p.exists():
            raise UnknownNetwork(f"no architecture file at {p}")
        fields, rows = parse_net_text(p.read_text(), str(p))
        return _assemble(fields["name"], fields, rows, str(p), input_hw)
    key = s.lower()
    if key not in _ARCH:
        raise UnknownNetwork(f"unknown network {source!r}; presets: "
                             f"{', '.join(network_preset_names())}")
    fields, rows = _ARCH[key]
    return _assemble(key, fields, rows, key, input_hw)


def parse_plan(text: str, net: NetworkSpec, paradigm: Paradigm) -> GranularityPlan:
    """Dash plan "4-2-2-1" validated against the network (`zoo.py:244-270`)."""
    try:
        values = tuple(int(p) for p in text.split("-"))
    except ValueError as exc:
        raise PlanLengthMismatch(f"bad plan {text!r}: {exc}") from exc
    if len(values) != len(net.stages):
        raise PlanLengthMismatch(f"plan {text!r} has {len(values)} entries, "
                                 f"network has {len(net.stages)} stages")
    if any(v < 1 for v in values):
        raise PlanLengthMismatch(f"plan {text!r} has non-positive entries")
    for si, v in enumerate(values, start=1):
        if paradigm is Paradigm.SPATIAL:
            f = net.stage_feature(si)
            if f.height % v or f.width % v:
                raise GranularityMismatch(f"stage {si}: S={v} does not divide "
                                          f"{f.height}x{f.width}")
        elif paradigm is Paradigm.CHANNEL:
            width = net.template_block(si).conv2.out_channels
            if width % v:
                raise GranularityMismatch(f"stage {si}: G={v} does not divide width {width}")
    return GranularityPlan(paradigm, values)


def config_for_stage(net: NetworkSpec, stage: int, paradigm: Paradigm,
                     plan: Optional[GranularityPlan]) -> DynamicConfig:
    """Per-stage DynamicConfig (`zoo.py:281-291`)."""
    if paradigm is Paradigm.SPATIAL:
        if plan is None:
            raise GranularityMismatch("spatial paradigm needs a plan")
        return DynamicConfig(paradigm, spatial_granularity=plan.values[stage - 1])
    if paradigm is Paradigm.CHANNEL:
        g = 1 if plan is None else plan.values[stage - 1]
        return DynamicConfig(paradigm, channel_granularity=g)
    return DynamicConfig(paradigm)

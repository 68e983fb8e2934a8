"""Configuration types of the dynamic-inference path.

Behavioural mirror of the block/config half of ``dynlat.core``
(`pkg/src/dynlat/core.py:41-52` Paradigm, `100-114` TensorShape,
`117-149` ConvLayerSpec, `152-199` BlockSpec, `202-224` DynamicConfig,
`227-255` ActivationProfile, `258-299` profile_for / enumerate_granularities /
validate_config).  Same field names, defaults, validation rules and error
classes, so a ``BlockSpec`` built for the reference is accepted verbatim.

The hardware-model half of ``dynlat.core`` (HardwareSpec, ``.hw`` files) is
the analytical latency predictor and is out of scope.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass
from typing import Optional

from .errors import GranularityMismatch, ParadigmFieldMissing, ShapeMismatch


class Paradigm(enum.Enum):
    """Which dynamic-inference scheme a block runs (`core.py:41-52`)."""

    SPATIAL = "spatial"
    CHANNEL = "channel"
    LAYER = "layer"
    STATIC = "static"


@dataclass(frozen=True)
class TensorShape:
    """C x H x W of one feature map, batch kept apart (`core.py:100-114`)."""

    channels: int
    height: int
    width: int

    def __post_init__(self):
        if self.channels < 1 or self.height < 1 or self.width < 1:
            raise ValueError("all dims must be >= 1")

    @property
    def elements(self) -> int:
        return self.channels * self.height * self.width


@dataclass(frozen=True)
class ConvLayerSpec:
    """One convolution; padding is always kernel//2 (`core.py:117-149`)."""

    in_channels: int
    out_channels: int
    kernel: int
    stride: int = 1
    groups: int = 1
    has_bias: bool = False

    def __post_init__(self):
        if self.in_channels < 1 or self.out_channels < 1:
            raise ValueError("channel counts must be positive")
        if self.kernel < 1 or self.kernel % 2 == 0:
            raise ValueError("kernel must be a positive odd integer")
        if self.stride not in (1, 2):
            raise ValueError("stride must be 1 or 2")
        if self.groups < 1:
            raise ValueError("groups must be positive")
        if self.in_channels % self.groups or self.out_channels % self.groups:
            raise ShapeMismatch(
                f"channels {self.in_channels}/{self.out_channels} not divisible "
                f"by groups {self.groups}"
            )

    def out_hw(self, h: int, w: int) -> tuple[int, int]:
        pad = self.kernel // 2
        return ((h + 2 * pad - self.kernel) // self.stride + 1,
                (w + 2 * pad - self.kernel) // self.stride + 1)


@dataclass(frozen=True)
class BlockSpec:
    """Bottleneck 1x1 -> 3x3 -> 1x1 with the stride on conv2 (`core.py:152-199`)."""

    conv1: ConvLayerSpec
    conv2: ConvLayerSpec
    conv3: ConvLayerSpec
    input_shape: TensorShape
    se_reduction: Optional[int] = None
    has_downsample: bool = False

    def __post_init__(self):
        c1, c2, c3 = self.conv1, self.conv2, self.conv3
        if c1.kernel != 1 or c3.kernel != 1:
            raise ShapeMismatch("conv1 and conv3 must be 1x1")
        if c2.kernel != 3:
            raise ShapeMismatch("conv2 must be 3x3")
        if c1.stride != 1 or c3.stride != 1:
            raise ShapeMismatch("block stride must live on conv2")
        if c1.out_channels != c2.in_channels:
            raise ShapeMismatch("conv1.out must equal conv2.in")
        if c2.out_channels != c3.in_channels:
            raise ShapeMismatch("conv2.out must equal conv3.in")
        if c1.in_channels != self.input_shape.channels:
            raise ShapeMismatch("conv1.in must match the input shape")
        if self.se_reduction is not None and self.se_reduction < 1:
            raise ValueError("se_reduction must be positive")
        if self.stride > 1 and not self.has_downsample:
            raise ShapeMismatch("a strided block needs a downsample path")

    @property
    def stride(self) -> int:
        return self.conv2.stride

    @property
    def output_shape(self) -> TensorShape:
        h, w = self.conv2.out_hw(self.input_shape.height, self.input_shape.width)
        return TensorShape(self.conv3.out_channels, h, w)

    @property
    def se_hidden(self) -> int:
        if self.se_reduction is None:
            return 0
        return max(1, self.conv2.out_channels // self.se_reduction)


@dataclass(frozen=True)
class DynamicConfig:
    """Paradigm plus granularity S (spatial) or G (channel) (`core.py:202-224`)."""

    paradigm: Paradigm
    spatial_granularity: Optional[int] = None
    channel_granularity: Optional[int] = None

    def __post_init__(self):
        if self.paradigm is Paradigm.SPATIAL and self.spatial_granularity is None:
            raise ParadigmFieldMissing("spatial paradigm requires spatial_granularity")
        if self.paradigm is Paradigm.CHANNEL and self.channel_granularity is None:
            raise ParadigmFieldMissing("channel paradigm requires channel_granularity")
        for g in (self.spatial_granularity, self.channel_granularity):
            if g is not None and g < 1:
                raise ValueError("granularities must be positive")


@dataclass(frozen=True)
class ActivationProfile:
    """Per-block activation rates (`core.py:227-255`)."""

    r_spatial: float = 1.0
    r_spatial_dilated: Optional[float] = None
    r_channel: float = 1.0
    r_layer: float = 1.0

    def __post_init__(self):
        for r in (self.r_spatial, self.r_channel, self.r_layer):
            if not 0.0 <= r <= 1.0:
                raise ValueError("activation rates must lie in [0, 1]")
        if self.r_spatial_dilated is not None:
            if not 0.0 <= self.r_spatial_dilated <= 1.0:
                raise ValueError("activation rates must lie in [0, 1]")
            if self.r_spatial_dilated < self.r_spatial:
                raise ValueError("r_spatial_dilated must be >= r_spatial")

    def dilated_or_default(self, granularity: int) -> float:
        if self.r_spatial_dilated is not None:
            return self.r_spatial_dilated
        return min(1.0, self.r_spatial * ((granularity + 2) / granularity) ** 2)


def profile_for(paradigm: Paradigm, rate: float) -> ActivationProfile:
    """Profile carrying ``rate`` on the paradigm's own field (`core.py:258-266`)."""
    if paradigm is Paradigm.SPATIAL:
        return ActivationProfile(r_spatial=rate)
    if paradigm is Paradigm.CHANNEL:
        return ActivationProfile(r_channel=rate)
    if paradigm is Paradigm.LAYER:
        return ActivationProfile(r_layer=rate)
    return ActivationProfile()


def enumerate_granularities(feature_size: int) -> tuple[int, ...]:
    """All divisors of a square feature side, ascending (`core.py:269-277`)."""
    if feature_size < 1:
        raise ValueError("feature_size must be >= 1")
    return tuple(d for d in range(1, feature_size + 1) if feature_size % d == 0)


def validate_config(block: BlockSpec, cfg: DynamicConfig) -> DynamicConfig:
    """Reject S/G that do not divide what they govern (`core.py:280-299`)."""
    out = block.output_shape
    if cfg.paradigm is Paradigm.SPATIAL:
        s = cfg.spatial_granularity
        if out.height % s or out.width % s:
            raise GranularityMismatch(
                f"S={s} does not divide the {out.height}x{out.width} output feature")
    elif cfg.paradigm is Paradigm.CHANNEL:
        g = cfg.channel_granularity
        if block.conv2.out_channels % g:
            raise GranularityMismatch(
                f"G={g} does not divide conv2 width {block.conv2.out_channels}")
    return cfg

"""Model parameter layouts.

Every model is a flat fp32 parameter vector on the device with named views.
``lr`` is the reference's multinomial logistic regression (fedsim/trainer.py:
45-59): entries ``weights`` [C, F] and ``bias`` [C].  ``cnn`` is the 2-layer
FEMNIST CNN of BASELINE config 2 (absent from the reference):
conv5x5(1->32)-relu-maxpool2-conv5x5(32->64)-relu-maxpool2-fc(3136->512)-relu-
fc(512->C), 'same' padding, P = 1,690,046 at C = 62.  ``resnet`` is the
CIFAR ResNet-18 with GroupNorm of BASELINE config 4 (also absent from the
reference), P = 11,173,962 at C = 10 (``resnet_layout``).  The CNN's tensors
use the channels-last layouts the kernels consume:

    conv1_w [32, 5, 5, 1]   conv1_b [32]
    conv2_w [64, 5, 5, 32]  conv2_b [64]
    fc1_w   [512, 3136]     (input index = (y*7 + x)*64 + c, NHWC flatten)
    fc1_b   [512]
    fc2_w   [C, 512]        fc2_b   [C]
"""

from __future__ import annotations

from dataclasses import dataclass
from math import prod

import numpy as np


@dataclass(frozen=True)
class ModelSpec:
    kind: str
    names: tuple[str, ...]
    shapes: tuple[tuple[int, ...], ...]
    n_features: int
    n_classes: int

    @property
    def sizes(self) -> tuple[int, ...]:
        return tuple(int(prod(s)) for s in self.shapes)

    @property
    def offsets(self) -> tuple[int, ...]:
        return tuple(int(v) for v in np.concatenate([[0], np.cumsum(self.sizes)[:-1]]))

    @property
    def numel(self) -> int:
        return int(sum(self.sizes))

    def columns(self):
        """(name, offset, size, shape) per entry, in flat order."""
        return list(zip(self.names, self.offsets, self.sizes, self.shapes))


def lr_spec(n_classes: int, n_features: int) -> ModelSpec:
    return ModelSpec("lr", ("weights", "bias"), ((n_classes, n_features), (n_classes,)),
                     n_features, n_classes)


CNN_C1, CNN_C2, CNN_H1, CNN_IMG = 32, 64, 512, 28


def cnn_spec(n_classes: int = 62) -> ModelSpec:
    flat = 7 * 7 * CNN_C2
    return ModelSpec(
        "cnn",
        ("conv1_w", "conv1_b", "conv2_w", "conv2_b", "fc1_w", "fc1_b", "fc2_w", "fc2_b"),
        ((CNN_C1, 5, 5, 1), (CNN_C1,), (CNN_C2, 5, 5, CNN_C1), (CNN_C2,), (CNN_H1, flat),
         (CNN_H1,), (n_classes, CNN_H1), (n_classes,)),
        CNN_IMG * CNN_IMG, n_classes)


def cnn_init(spec: ModelSpec, seed: int = 0) -> np.ndarray:
    """Deterministic initialisation with PyTorch's default Conv2d/Linear rule
    (weights and biases ~ U(-1/sqrt(fan_in), 1/sqrt(fan_in))), as the FedML
    FEMNIST CNN uses; float32 flat vector.  The reference has no CNN, so the
    init is the builder's choice."""
    g = np.random.default_rng([seed, 97])
    out = np.zeros(spec.numel, dtype=np.float32)
    fan_in = {"conv1": 25, "conv2": 800, "fc1": 3136, "fc2": 512}
    for name, off, size, _ in spec.columns():
        bound = 1.0 / np.sqrt(fan_in[name.split("_")[0]])
        out[off:off + size] = g.uniform(-bound, bound, size).astype(np.float32)
    return out


RESNET_PLANES = (64, 128, 256, 512)
RESNET_GN_GROUPS = 2


def resnet_layout(n_classes: int = 10):
    """[(name, shape)] of the CIFAR ResNet-18 with GroupNorm (BASELINE config
    4), flat order: conv1, gn1, then per stage l1..l4 and block 0/1
    conv1/gn1/conv2/gn2 (+ down/down_gn on the first block of stages 2-4),
    then fc.  Conv weights are [co][kh][kw][ci] (channels-last)."""
    out = [("conv1_w", (64, 3, 3, 3)), ("gn1_w", (64,)), ("gn1_b", (64,))]
    cin = 64
    for li, planes in enumerate(RESNET_PLANES, start=1):
        for bi in range(2):
            p = f"l{li}.{bi}."
            out += [(p + "conv1_w", (planes, 3, 3, cin)), (p + "gn1_w", (planes,)), (p + "gn1_b", (planes,)),
                    (p + "conv2_w", (planes, 3, 3, planes)), (p + "gn2_w", (planes,)),
                    (p + "gn2_b", (planes,))]
            if bi == 0 and li > 1:
                out += [(p + "down_w", (planes, 1, 1, cin)), (p + "down_gn_w", (planes,)),
                        (p + "down_gn_b", (planes,))]
            cin = planes
    out += [("fc_w", (n_classes, 512)), ("fc_b", (n_classes,))]
    return out


def resnet_spec(n_classes: int = 10) -> ModelSpec:
    """ResNet-18 (GroupNorm, 2 groups), CIFAR variant: P = 11,173,962 at 10
    classes.  Inputs: 3072 features = a 32x32x3 NHWC image."""
    lay = resnet_layout(n_classes)
    return ModelSpec("resnet", tuple(n for n, _ in lay), tuple(s for _, s in lay), 32 * 32 * 3, n_classes)


def resnet_init(spec: ModelSpec, seed: int = 0) -> np.ndarray:
    """PyTorch's default rules: conv/fc weights ~ U(-1/sqrt(fan_in),
    1/sqrt(fan_in)), fc bias likewise, GroupNorm weight 1 and bias 0;
    deterministic per seed (float32 flat vector)."""
    g = np.random.default_rng([seed, 98])
    out = np.zeros(spec.numel, dtype=np.float32)
    for name, off, size, shape in spec.columns():
        if "gn" in name:
            out[off:off + size] = 1.0 if name.endswith("_w") else 0.0
            continue
        fan_in = int(np.prod(shape[1:])) if name != "fc_b" else 512
        bound = 1.0 / np.sqrt(fan_in)
        out[off:off + size] = g.uniform(-bound, bound, size).astype(np.float32)
    return out


def init_params(spec: ModelSpec, seed: int = 0) -> np.ndarray:
    if spec.kind == "resnet":
        return resnet_init(spec, seed)
    return cnn_init(spec, seed)


def spec_for(kind: str, n_features: int, n_classes: int) -> ModelSpec:
    if kind == "lr":
        return lr_spec(n_classes, n_features)
    if kind == "cnn":
        if n_features != CNN_IMG * CNN_IMG:
            raise ValueError(f"cnn needs 28x28 inputs, got {n_features} features")
        return cnn_spec(n_classes)
    if kind == "resnet":
        if n_features != 32 * 32 * 3:
            raise ValueError(f"resnet needs 32x32x3 inputs, got {n_features} features")
        return resnet_spec(n_classes)
    raise ValueError(f"unknown model kind {kind!r}")

"""Model parameter layouts.

Every model is a flat fp32 parameter vector on the device with named views.
``lr`` is the reference's multinomial logistic regression (fedsim/trainer.py:
45-59): entries ``weights`` [C, F] and ``bias`` [C].  ``cnn`` is the 2-layer
FEMNIST CNN of BASELINE config 2 (absent from the reference):
conv5x5(1->32)-relu-maxpool2-conv5x5(32->64)-relu-maxpool2-fc(3136->512)-relu-
fc(512->C), 'same' padding, P = 1,690,046 at C = 62.  Its tensors use the
channels-last layouts the kernels consume:

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


def spec_for(kind: str, n_features: int, n_classes: int) -> ModelSpec:
    if kind == "lr":
        return lr_spec(n_classes, n_features)
    if kind == "cnn":
        if n_features != CNN_IMG * CNN_IMG:
            raise ValueError(f"cnn needs 28x28 inputs, got {n_features} features")
        return cnn_spec(n_classes)
    raise ValueError(f"unknown model kind {kind!r}")

"""Workload generators: the reference's ``random_spec`` property-test sampler
(workloads.py:111-142), seeded integer operands (simulator.py:445-455), and
the BASELINE.json configurations including the 53-layer ResNet-50 v1.5 sweep
(SURVEY.md Appendix A).  Synthetic data only: the paper evaluates on
ImageNet-resolution inference, which seeded N(0,1) activations at the same
shapes stand in for.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import ConvSpec, Layout, ShapeError, Tensor


def random_spec(rng: np.random.Generator, *, max_hw: int = 16, max_n: int = 8, max_co: int = 16,
                max_f: int = 5, max_stride: int = 4, max_pad: int = 2, max_dilation: int = 2,
                c_i_choices=(1, 2, 3, 8, 16, 128)) -> ConvSpec:
    """A valid random layer inside the bounds; same sampling sequence as the
    reference (workloads.py:111-142) so a seed yields the same specs."""
    while True:
        f_h, f_w = (int(rng.integers(1, max_f + 1)) for _ in range(2))
        d_h, d_w = (int(rng.integers(1, max_dilation + 1)) for _ in range(2))
        p_h, p_w = (int(rng.integers(0, max_pad + 1)) for _ in range(2))
        need_h = max(1, d_h * (f_h - 1) + 1 - 2 * p_h)
        need_w = max(1, d_w * (f_w - 1) + 1 - 2 * p_w)
        if need_h > max_hw or need_w > max_hw:
            continue
        try:
            return ConvSpec(n=int(rng.integers(1, max_n + 1)), c_i=int(rng.choice(c_i_choices)),
                            h_i=int(rng.integers(need_h, max_hw + 1)), w_i=int(rng.integers(need_w, max_hw + 1)),
                            c_o=int(rng.integers(1, max_co + 1)), h_f=f_h, w_f=f_w,
                            stride_h=int(rng.integers(1, max_stride + 1)),
                            stride_w=int(rng.integers(1, max_stride + 1)),
                            pad_h=p_h, pad_w=p_w, dilation_h=d_h, dilation_w=d_w)
        except ShapeError:
            continue


def default_operands(spec: ConvSpec, seed: int = 0):
    """Seeded integer IFMap/filters in [-4, 4] (simulator.py:445-455)."""
    rng = np.random.default_rng(seed)
    x = rng.integers(-4, 5, size=(spec.n, spec.h_i, spec.w_i, spec.c_i)).astype(np.int64)
    f = rng.integers(-4, 5, size=(spec.h_f, spec.w_f, spec.c_i, spec.c_o)).astype(np.int64)
    return Tensor.from_array(x, Layout.NHWC), Tensor.from_array(f, Layout.HWCN)


@dataclass(frozen=True)
class Layer:
    name: str
    spec: ConvSpec
    dtype: str = "bf16"          # compute dtype: bf16 | int8
    relu_input: bool = False     # inputs clamped at 0 (post-ReLU activations)


def resnet50_layers(n: int = 256) -> list:
    """The 53 convolutions of ResNet-50 v1.5 at 224x224:
    7x7/2 stem with C=3 zero-padded to 8, then bottlenecks 1x1 -> 3x3 (stride
    on the 3x3) -> 1x1, plus a 1x1 projection in each stage's first block."""
    layers = [Layer("stem", ConvSpec.square(n, 8, 224, 64, 7, stride=2, pad=3))]
    hw, c_in = 56, 64  # after the 3x3/2 max-pool
    for stage, (width, blocks) in enumerate(zip((64, 128, 256, 512), (3, 4, 6, 3)), start=2):
        for b in range(blocks):
            stride = 2 if (b == 0 and stage > 2) else 1
            out_hw = hw // stride
            tag = f"s{stage}b{b}"
            layers.append(Layer(f"{tag}_1x1a", ConvSpec.square(n, c_in, hw, width, 1), relu_input=b > 0))
            layers.append(Layer(f"{tag}_3x3", ConvSpec.square(n, width, hw, width, 3, stride=stride, pad=1),
                                relu_input=True))
            layers.append(Layer(f"{tag}_1x1b", ConvSpec.square(n, width, out_hw, 4 * width, 1), relu_input=True))
            if b == 0:
                layers.append(Layer(f"{tag}_proj", ConvSpec.square(n, c_in, hw, 4 * width, 1, stride=stride)))
            c_in, hw = 4 * width, out_hw
    return layers


def baseline_configs() -> dict:
    """BASELINE.json `configs`, keyed cfg1..cfg5 (cfg4 = the ResNet-50 sweep)."""
    return {
        "cfg1": [Layer("cfg1_3x3_s1", ConvSpec.square(8, 64, 56, 64, 3, stride=1, pad=1))],
        "cfg2": [Layer("cfg2a_3x3_s2", ConvSpec.square(32, 128, 56, 128, 3, stride=2, pad=1), relu_input=True),
                 Layer("cfg2b_1x1_s2", ConvSpec.square(32, 256, 56, 512, 1, stride=2, pad=0), relu_input=True)],
        "cfg3": [Layer("cfg3_3x3_d2", ConvSpec.square(16, 512, 64, 512, 3, stride=1, pad=2, dilation=2))],
        "cfg4": resnet50_layers(256),
        "cfg5": [Layer("cfg5_i8_s1", ConvSpec.square(64, 256, 28, 256, 3, stride=1, pad=1), dtype="int8"),
                 Layer("cfg5_i8_s2", ConvSpec.square(64, 256, 28, 256, 3, stride=2, pad=1), dtype="int8"),
                 Layer("cfg5_i8_d2", ConvSpec.square(64, 256, 28, 256, 3, stride=1, pad=2, dilation=2),
                       dtype="int8")],
    }


def synthetic_operands(layer: Layer, seed: int = 0, n: int | None = None, device=None):
    """Seeded operands with BASELINE.json value distributions.

    bf16 layers: activations N(0,1) (clamped at 0 when post-ReLU), weights
    Kaiming-normal std sqrt(2/(C*R*S)); fp32 draws rounded to bf16.
    int8 layers: uniform integers in [-128, 127].
    Returns torch tensors (x NHWC, w HWCN) on ``device`` (default CPU).
    For the stem, channels 3..7 of both operands are zero (C=3 padded to 8).
    """
    import torch

    sp = layer.spec if n is None else layer.spec.with_batch(n)
    g = torch.Generator(device="cpu").manual_seed(seed)
    xs = (sp.n, sp.h_i, sp.w_i, sp.c_i)
    ws = (sp.h_f, sp.w_f, sp.c_i, sp.c_o)
    if layer.dtype == "int8":
        x = torch.randint(-128, 128, xs, generator=g, dtype=torch.int16).to(torch.int8)
        w = torch.randint(-128, 128, ws, generator=g, dtype=torch.int16).to(torch.int8)
    else:
        x = torch.randn(xs, generator=g, dtype=torch.float32)
        if layer.relu_input:
            x.clamp_(min=0)
        std = (2.0 / (sp.c_i * sp.h_f * sp.w_f)) ** 0.5
        w = torch.randn(ws, generator=g, dtype=torch.float32) * std
        if layer.name == "stem":
            x[..., 3:] = 0
            w[:, :, 3:, :] = 0
        x, w = x.to(torch.bfloat16), w.to(torch.bfloat16)
    if device is not None:
        x, w = x.to(device), w.to(device)
    return x, w


__all__ = ["Layer", "baseline_configs", "default_operands", "random_spec", "resnet50_layers",
           "synthetic_operands"]

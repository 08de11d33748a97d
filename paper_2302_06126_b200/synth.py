"""Seeded synthetic inputs shaped like the paper's workloads.

This module is shared by the tests, bench.py and smoke(); it holds NONE of the method's
arithmetic (no products, sums, scales or casts of the SFB path) — only random draws, so both the
CUDA path and the oracle can be fed the same arrays.

Seeds: numpy Generator(PCG64(SeedSequence([230206126, config_id, layer_id, rank, tensor_id]))),
tensor_id 0 = X, 1 = dY, 2 = W0, 3 = v0. Values are drawn in fp32; bf16 configs
are rounded to bf16 by the consumer (torch RNE) before either side sees them.

Value structure (Table "tab:models" P:693-700 workloads):
  post-ReLU activations (~50% zeros) feeding VGG/AlexNet FC layers, ReLU-masked small backward
  gradients N(0, 1e-3^2)*Bernoulli(0.5), classifier gradients softmax(z) - onehot(y), LayerNorm-like
  N(0,1) / GELU / tanh-pooled inputs for Transformer and BERT layers, and an exactness suite of
  small integers in {-3..3}.
"""
from dataclasses import dataclass, field

import numpy as np

SEED_ROOT = 230206126
T_X, T_DY, T_W, T_V = 0, 1, 2, 3


@dataclass(frozen=True)
class Layer:
    name: str
    M: int          # input features (H1)
    N: int          # output features (H2)
    B: int          # rows per replica
    x_dist: str
    dy_dist: str


@dataclass(frozen=True)
class Config:
    cid: int
    name: str
    layers: tuple
    ns: tuple                  # replica counts the config is quoted at
    in_dtype: str = "bf16"     # "f32" | "bf16"
    wire_dtype: str = "bf16"
    out_dtype: str = "f32"
    sgd: dict = field(default=None)


_VGG_FC = (
    Layer("fc6", 25088, 4096, 32, "relu", "masked_small"),
    Layer("fc7", 4096, 4096, 32, "relu", "masked_small"),
    Layer("fc8", 4096, 1000, 32, "relu", "softmax_onehot"),
)

CONFIGS = {
    1: Config(1, "toy_fc_64x32", (Layer("fc", 64, 32, 4, "normal", "normal"),), (2,),
              "f32", "f32", "f32"),
    2: Config(2, "vgg19_fc", _VGG_FC, (1, 2, 4, 8)),
    3: Config(3, "alexnet_vgg16_fc", (
        Layer("alexnet_fc6", 9216, 4096, 64, "relu", "masked_small"),
        Layer("alexnet_fc7", 4096, 4096, 64, "relu", "masked_small"),
        Layer("alexnet_fc8", 4096, 1000, 64, "relu", "softmax_onehot"),
        Layer("vgg16_fc6", 25088, 4096, 64, "relu", "masked_small"),
        Layer("vgg16_fc7", 4096, 4096, 64, "relu", "masked_small"),
        Layer("vgg16_fc8", 4096, 1000, 64, "relu", "softmax_onehot"),
    ), (1, 2, 4, 8)),
    4: Config(4, "transformer_base", (
        Layer("out_proj", 512, 32000, 256, "normal", "softmax_onehot"),
        Layer("ffn1", 512, 2048, 256, "normal", "small"),
        Layer("ffn2", 2048, 512, 256, "gelu", "small"),
    ), (1, 2, 4, 8)),
    5: Config(5, "bert_large", (
        Layer("ffn1", 1024, 4096, 128, "normal", "small"),
        Layer("ffn2", 4096, 1024, 128, "gelu", "small"),
        Layer("pooler", 1024, 1024, 2, "tanh", "small"),
    ), (8,), sgd=dict(lr=1e-3, momentum=0.9, weight_decay=0.0)),
}


def rng(config_id, layer_id, rank, tensor_id):
    return np.random.Generator(np.random.PCG64(
        np.random.SeedSequence([SEED_ROOT, config_id, layer_id, rank, tensor_id])))


def _gelu_tanh(x):
    return 0.5 * x * (1.0 + np.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


def draw(dist, rows, cols, g):
    """rows x cols float32 sample of the named distribution."""
    if dist == "normal":
        a = g.standard_normal((rows, cols), dtype=np.float32)
    elif dist == "relu":
        a = np.maximum(g.standard_normal((rows, cols), dtype=np.float32), 0)
    elif dist == "gelu":
        a = _gelu_tanh(g.standard_normal((rows, cols), dtype=np.float32))
    elif dist == "tanh":
        a = np.tanh(g.standard_normal((rows, cols), dtype=np.float32))
    elif dist == "small":
        a = g.standard_normal((rows, cols), dtype=np.float32) * np.float32(1e-3)
    elif dist == "masked_small":
        a = g.standard_normal((rows, cols), dtype=np.float32) * np.float32(1e-3)
        a *= (g.random((rows, cols), dtype=np.float32) < 0.5)
    elif dist == "softmax_onehot":
        z = g.standard_normal((rows, cols), dtype=np.float32)
        e = np.exp(z - z.max(axis=1, keepdims=True))
        a = e / e.sum(axis=1, keepdims=True)
        y = g.integers(0, cols, size=rows)
        a[np.arange(rows), y] -= 1.0
    elif dist == "int3":
        a = g.integers(-3, 4, size=(rows, cols)).astype(np.float32)
    elif dist == "ones":
        a = np.ones((rows, cols), dtype=np.float32)
    else:
        raise ValueError(dist)
    return np.ascontiguousarray(a, dtype=np.float32)


def factors(config_id, layer_id, rank, M, N, B, x_dist, dy_dist):
    """(X_r, dY_r) float32 for one replica: B x M and B x N."""
    X = draw(x_dist, B, M, rng(config_id, layer_id, rank, T_X))
    dY = draw(dy_dist, B, N, rng(config_id, layer_id, rank, T_DY))
    return X, dY


def all_factors(config_id, layer_id, n, M, N, B, x_dist, dy_dist):
    """Every replica's factors stacked replica-major: X (n, B, M), dY (n, B, N) float32."""
    Xs, dYs = zip(*(factors(config_id, layer_id, r, M, N, B, x_dist, dy_dist) for r in range(n)))
    return np.stack(Xs), np.stack(dYs)


def sgd_state(config_id, layer_id, M, N):
    """W0 ~ N(0, 0.02^2) and v0 = 0, float32, M x N."""
    W = rng(config_id, layer_id, 0, T_W).standard_normal((M, N), dtype=np.float32) * np.float32(0.02)
    return np.ascontiguousarray(W), np.zeros((M, N), dtype=np.float32)

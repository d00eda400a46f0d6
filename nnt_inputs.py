"""Seeded synthetic inputs shared by the oracle-side tests and the CUDA-side tests/bench.

This module holds NO arithmetic of the method: only configurations and
random-number generation (NumPy PCG64).  Both sides draw their inputs from here
so that parity tests compare the two implementations on identical data.

Recipe:
  * x  ~ N(0, 1) fp32 [N_b, N_s, N_e]; sequence j of the global batch is drawn
    from SeedSequence([seed, j]) so a rank's batch tiles are bit-identical to
    the same tiles of a 1-GPU run.
  * r  ~ N(0, 1) fp32 (linear-probe loss direction; dy = r / T_global).
  * parameters: "parity" init (weights N(0, 1/fan_in), biases N(0, 0.1^2),
    gamma ~ 1 + N(0, 0.1^2), beta ~ N(0, 0.1^2)) so softmax and GELU are
    exercised non-trivially; "gpt2" init (N(0, 0.02^2), proj N(0,(0.02/sqrt(2L))^2),
    zero biases, gamma = 1, beta = 0) for throughput runs (reading R16).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

PARAM_NAMES = ("ln1_g", "ln1_b", "w_qkv", "b_qkv", "w_o", "b_o",
               "ln2_g", "ln2_b", "w_fc", "b_fc", "w_pr", "b_pr")


@dataclasses.dataclass(frozen=True)
class BlockConfig:
    name: str
    L: int       # layers
    E: int       # N_e, embedding size
    H: int       # N_h, heads
    S: int       # N_s, sequence length
    B: int       # N_b, per-GPU batch (sequences)
    tile: int    # logical tile along embedding / hidden / sequence axes
    dtype: str   # "f32" or "bf16"

    @property
    def Dh(self):
        return self.E // self.H

    @property
    def F(self):
        return 4 * self.E

    @property
    def T(self):
        return self.B * self.S


# BASELINE.json configs.
CONFIGS = {
    "tiny": BlockConfig("tiny", 1, 64, 2, 32, 2, 16, "f32"),
    "small": BlockConfig("small", 12, 768, 12, 1024, 8, 1024, "bf16"),
    "large": BlockConfig("large", 36, 1280, 20, 1024, 8, 1024, "bf16"),
    "xl": BlockConfig("xl", 48, 1600, 25, 1024, 8, 1024, "bf16"),
    "wide": BlockConfig("wide", 1, 8192, 128, 1024, 8, 1024, "bf16"),
}


def param_shapes(E):
    F = 4 * E
    return {
        "ln1_g": (E,), "ln1_b": (E,),
        "w_qkv": (3 * E, E), "b_qkv": (3 * E,),
        "w_o": (E, E), "b_o": (E,),
        "ln2_g": (E,), "ln2_b": (E,),
        "w_fc": (F, E), "b_fc": (F,),
        "w_pr": (E, F), "b_pr": (E,),
    }


def _rng(*key):
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(list(key))))


def make_params(E, seed=1234, layer=0, init="parity", n_layers=1):
    """One block's parameters as fp32 arrays (dict keyed by PARAM_NAMES)."""
    shapes = param_shapes(E)
    out = {}
    for i, name in enumerate(PARAM_NAMES):
        rng = _rng(seed, layer, i)
        shp = shapes[name]
        if init == "parity":
            if name.startswith("w_"):
                a = rng.standard_normal(shp) / math.sqrt(shp[1])
            elif name.endswith("_g"):
                a = 1.0 + 0.1 * rng.standard_normal(shp)
            else:
                a = 0.1 * rng.standard_normal(shp)
        elif init == "gpt2":
            if name.startswith("w_"):
                std = 0.02 / math.sqrt(2 * n_layers) if name in ("w_o", "w_pr") else 0.02
                a = std * rng.standard_normal(shp, dtype=np.float32)
            elif name.endswith("_g"):
                a = np.ones(shp)
            else:
                a = np.zeros(shp)
        else:
            raise ValueError(init)
        out[name] = np.ascontiguousarray(a, dtype=np.float32)
    return out


def make_x(E, S, batch_begin, batch_end, seed=5678, scale=1.0):
    """Input activations for global sequences [batch_begin, batch_end): fp32 [n, S, E]."""
    seqs = [(scale * _rng(seed, 0, j).standard_normal((S, E), dtype=np.float32))
            for j in range(batch_begin, batch_end)]
    return np.ascontiguousarray(np.stack(seqs).astype(np.float32))


def make_r(E, S, batch_begin, batch_end, seed=5678):
    """Probe-loss directions r for global sequences [batch_begin, batch_end)."""
    seqs = [_rng(seed, 1, j).standard_normal((S, E), dtype=np.float32)
            for j in range(batch_begin, batch_end)]
    return np.ascontiguousarray(np.stack(seqs).astype(np.float32))


def make_matrix(shape, seed, kind="normal", lo=-4, hi=4):
    """Generic test matrix: 'normal' N(0,1) or 'int' uniform integers in [lo, hi]."""
    rng = _rng(seed, 7)
    if kind == "normal":
        return rng.standard_normal(shape).astype(np.float32)
    if kind == "int":
        return rng.integers(lo, hi + 1, size=shape).astype(np.float32)
    raise ValueError(kind)


# ---------------------------------------------------------------- GPT-2 shell
def make_shell_params(V, S_max, E, seed=1234, init="parity"):
    """Token table wte [V, E], position table wpe [S_max, E], final LayerNorm (lnf_g, lnf_b).

    parity: wte, wpe ~ N(0, 1/E), lnf_g ~ 1 + N(0, 0.1^2), lnf_b ~ N(0, 0.1^2);
    gpt2:   wte ~ N(0, 0.02^2), wpe ~ N(0, 0.01^2), lnf_g = 1, lnf_b = 0."""
    out = {}
    for i, (name, shp) in enumerate((("wte", (V, E)), ("wpe", (S_max, E)), ("lnf_g", (E,)), ("lnf_b", (E,)))):
        rng = _rng(seed, 999, i)
        if name in ("wte", "wpe"):
            std = (0.02 if name == "wte" else 0.01) if init == "gpt2" else 1.0 / math.sqrt(E)
            a = std * rng.standard_normal(shp, dtype=np.float32)
        elif name == "lnf_g":
            a = np.ones(shp) if init == "gpt2" else 1.0 + 0.1 * rng.standard_normal(shp)
        else:
            a = np.zeros(shp) if init == "gpt2" else 0.1 * rng.standard_normal(shp)
        out[name] = np.ascontiguousarray(a, dtype=np.float32)
    return out


def make_ids(V, S, batch_begin, batch_end, seed=5678):
    """Token ids ~ U[0, V) for global sequences [batch_begin, batch_end) (int32 [n, S + 1]):
    inputs are [:, :S], next-token labels [:, 1:]."""
    seqs = [_rng(seed, 2, j).integers(0, V, size=S + 1, dtype=np.int64) for j in range(batch_begin, batch_end)]
    return np.ascontiguousarray(np.stack(seqs).astype(np.int32))

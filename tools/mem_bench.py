"""Times the HBM-bound libnnt kernels of one GPT-2 block (LayerNorm fwd/bwd, bias-gradient
column sums, attention row-dot, probe loss) through the C ABI: back-to-back launches replayed
from a CUDA graph, median of several rounds; GB/s from the algorithmic bytes of each call
(inputs of 25-50 MB stay partly L2-resident across repeats: an optimistic bound).

    python tools/mem_bench.py [--config small] [--only ln_fwd,ln_bwd,...]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2504_13236_b200 import nnt  # noqa: E402


def timeit(fn, reps=20, rounds=5):
    """reps launches captured in one CUDA graph (host launch cost excluded, as in the bench's
    graph-replayed step), timed over `rounds` replays; median per launch in us."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(rounds):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / reps)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="small")
    ap.add_argument("--only", default=None)
    a = ap.parse_args()
    L, E, H, S, B = bench.CONFIGS[a.config]
    T, F, Dh = B * S, 4 * E, E // H
    f32 = dict(device="cuda", dtype=torch.float32)
    bf = dict(device="cuda", dtype=torch.bfloat16)
    x = torch.randn(T, E, **f32)
    dy = torch.randn(T, E, **f32)
    dres = torch.randn(T, E, **f32)
    dx = torch.empty(T, E, **f32)
    dx16 = torch.empty(T, E, **bf)
    h = torch.empty(T, E, **bf)
    g = torch.ones(E, **f32)
    b = torch.zeros(E, **f32)
    mean = torch.empty(T, **f32)
    rstd = torch.empty(T, **f32)
    nnt.nnt_layernorm_fwd(x, T, E, E, 1024, g, b, 1e-5, h, nnt.NNT_BF16, E, mean, rstd)
    lscr = torch.empty(nnt.nnt_layernorm_bwd_scratch_bytes(T, E), device="cuda", dtype=torch.uint8)
    dg = torch.zeros(E, **f32)
    db = torch.zeros(F, **f32)
    du = torch.randn(T, F, **bf)
    dqkv = torch.randn(T, 3 * E, **bf)
    cscr = torch.empty(nnt.nnt_bias_grad_scratch_bytes(T, F), device="cuda", dtype=torch.uint8)
    dO = torch.randn(T, E, **bf)
    O = torch.randn(T, E, **bf)
    D = torch.empty(B * H * S, **f32)
    loss = torch.zeros(1, **f32)
    dscr = torch.empty(nnt.nnt_dot_scratch_bytes(T * E), device="cuda", dtype=torch.uint8)
    cases = {
        "ln_fwd": (lambda: nnt.nnt_layernorm_fwd(x, T, E, E, 1024, g, b, 1e-5, h, nnt.NNT_BF16, E, mean, rstd),
                   T * E * (4 + 2) + 8 * T),
        "ln_bwd": (lambda: nnt.nnt_layernorm_bwd(dy, E, x, E, mean, rstd, g, T, E, dres, dx, E, dx16, dg, dg, None, 0,
                                                 lscr, lscr.numel()), T * E * (4 * 4 + 2) + 8 * T),
        "colsum_f32+copy": (lambda: nnt.nnt_bias_grad(dy, nnt.NNT_F32, T, E, E, db, 0, dx16, cscr, cscr.numel()),
                            T * E * 6),
        "colsum_f32": (lambda: nnt.nnt_bias_grad(dy, nnt.NNT_F32, T, E, E, db, 0, None, cscr, cscr.numel()),
                       T * E * 4),
        "colsum_bf16_4E": (lambda: nnt.nnt_bias_grad(du, nnt.NNT_BF16, T, F, F, db, 0, None, cscr, cscr.numel()),
                           T * F * 2),
        "colsum_bf16_3E": (lambda: nnt.nnt_bias_grad(dqkv, nnt.NNT_BF16, T, 3 * E, 3 * E, db, 0, None, cscr,
                                                     cscr.numel()), T * 3 * E * 2),
        "rowdot": (lambda: nnt.nnt_attn_rowdot(dO, O, nnt.NNT_BF16, B, S, H, Dh, D), T * E * 4),
        "dot": (lambda: nnt.nnt_dot(x, dy, T * E, 1.0, loss, dscr, dscr.numel()), T * E * 8),
        "scale": (lambda: nnt.nnt_scale(x, 0.5, dx, T * E), T * E * 8),
    }
    print(f"{'kernel':16s} {'us':>8s} {'GB/s':>8s}")
    for name, (fn, nbytes) in cases.items():
        if a.only and name not in a.only.split(","):
            continue
        us = timeit(fn)
        print(f"{name:16s} {us:8.1f} {nbytes / us / 1e3:8.1f}")


if __name__ == "__main__":
    main()

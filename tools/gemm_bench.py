"""Times every GEMM of one GPT-2 block (fwd + bwd) through nnt_tile_gemm.

    python tools/gemm_bench.py [--config small] [--iters 20]

Prints per-GEMM device time (CUDA events, median), TFLOP/s (executed FLOPs) and
GB/s (algorithmic bytes).  Inputs are random bf16; results are not checked here
(tests/test_gpu_gemm.py does that).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2504_13236_b200 import nnt  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="small")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--only", default=None, help="comma-separated GEMM names")
    ap.add_argument("--no-ws", action="store_true", help="no workspace for the unbatched GEMMs (no stream-K)")
    a = ap.parse_args()
    L, E, H, S, B = bench.CONFIGS[a.config]
    T, F, Dh = B * S, 4 * E, E // H
    bf = dict(device="cuda", dtype=torch.bfloat16)
    f32 = dict(device="cuda", dtype=torch.float32)
    h = torch.randn(T, 3 * E, **bf) * 0.1          # activations (also qkv / dqkv)
    g = torch.randn(T, F, **bf) * 0.1
    w = torch.randn(3 * E, F, **bf) * 0.02         # any weight view
    P = torch.randn(B, H, S, S, **bf) * 0.01
    outf = torch.empty(max(T * F, B * H * S * S), **f32)
    outb = torch.empty(max(T * F, B * H * S * S), **bf)
    aux = torch.randn(T, F, **bf)
    bias = torch.zeros(F, **f32)
    res = torch.zeros(T, E, **f32)
    bh = (B, H)
    es = 2
    big = torch.randn(8192, 8192, **bf) * 0.05
    spart = torch.empty(B * H * S * (S // 32) * 2, **f32)
    dvec = torch.zeros(B * H * S, **f32)
    rstats = torch.zeros(B * H * S * 2, **f32)
    rowsum = torch.zeros(F, **f32)
    cases = [
        # name, ta, tb, M, N, K, batch, A, lda, sa, B, ldb, sb, C, cdt, ldc, sc, epi, causal-frac
        ("qkv", 0, 1, T, 3 * E, E, None, h, E, None, w, E, None, outb, 1, 3 * E, None,
         nnt.make_epilogue(bias=bias), 1.0),
        ("scores", 0, 1, S, S, Dh, bh, h, 3 * E, (S * 3 * E, Dh), h.data_ptr() + es * E, 3 * E, (S * 3 * E, Dh),
         outf, 0, S, (H * S * S, S * S), nnt.make_epilogue(causal=1), 0.5),
        ("scores+stats", 0, 1, S, S, Dh, bh, h, 3 * E, (S * 3 * E, Dh), h.data_ptr() + es * E, 3 * E,
         (S * 3 * E, Dh), outf, 0, S, (H * S * S, S * S),
         nnt.make_epilogue(causal=1, row_stats=spart, ld_row_stats=S // 32), 0.5),
        ("rowstats", 0, 1, S, S, Dh, bh, h, 3 * E, (S * 3 * E, Dh), h.data_ptr() + es * E, 3 * E, (S * 3 * E, Dh),
         None, 0, S, (H * S * S, S * S), nnt.make_epilogue(causal=1, act=4, row_stats=rstats), 0.5),
        ("softmaxP", 0, 1, S, S, Dh, bh, h, 3 * E, (S * 3 * E, Dh), h.data_ptr() + es * E, 3 * E, (S * 3 * E, Dh),
         outb, 1, S, (H * S * S, S * S), nnt.make_epilogue(causal=1, act=5, row_stats=rstats), 0.5),
        ("dp_dA", 0, 1, S, S, Dh, bh, h, E, (S * E, Dh), h.data_ptr() + es * 2 * E, 3 * E, (S * 3 * E, Dh),
         outb, 1, S, (H * S * S, S * S),
         nnt.make_epilogue(causal=1, act=3, aux=P, ld_aux=S, rowvec=dvec, rowscale=0.125), 0.5),
        ("pv", 0, 0, S, Dh, S, bh, P, S, (H * S * S, S * S), h, 3 * E, (S * 3 * E, Dh), outb, 1, E, (S * E, Dh),
         nnt.make_epilogue(causal=2), 0.5),
        ("out", 0, 1, T, E, E, None, h, E, None, w, E, None, outf, 0, E, None,
         nnt.make_epilogue(bias=bias, residual=res, ld_residual=E), 1.0),
        ("fc+gelu", 0, 1, T, F, E, None, h, E, None, w, E, None, outb, 1, F, None,
         nnt.make_epilogue(bias=bias, act=1, aux=aux, ld_aux=F), 1.0),
        ("fc_plain", 0, 1, T, F, E, None, h, E, None, w, E, None, outb, 1, F, None, None, 1.0),
        ("proj_plain", 0, 1, T, E, F, None, g, F, None, w, F, None, outb, 1, E, None, None, 1.0),
        ("proj_dx_plain", 0, 0, T, F, E, None, h, E, None, w, F, None, outb, 1, F, None, None, 1.0),
        ("proj", 0, 1, T, E, F, None, g, F, None, w, F, None, outf, 0, E, None,
         nnt.make_epilogue(bias=bias, residual=res, ld_residual=E), 1.0),
        ("proj_dw", 1, 0, E, F, T, None, h, E, None, g, F, None, outf, 0, F, None, None, 1.0),
        ("proj_dx+gelu'", 0, 0, T, F, E, None, h, E, None, w, F, None, outb, 1, F, None,
         nnt.make_epilogue(act=2, aux=aux, ld_aux=F), 1.0),
        ("fc_dw", 1, 0, F, E, T, None, g, F, None, h, E, None, outf, 0, E, None, None, 1.0),
        ("fc_dx", 0, 0, T, E, F, None, g, F, None, w, E, None, outf, 0, E, None, None, 1.0),
        ("out_dw", 1, 0, E, E, T, None, h, E, None, h, E, None, outf, 0, E, None, None, 1.0),
        ("out_dx", 0, 0, T, E, E, None, h, E, None, w, E, None, outb, 1, E, None, None, 1.0),
        ("att_dp", 0, 1, S, S, Dh, bh, h, E, (S * E, Dh), h.data_ptr() + es * 2 * E, 3 * E, (S * 3 * E, Dh),
         outf, 0, S, (H * S * S, S * S), nnt.make_epilogue(causal=1), 0.5),
        ("att_dv", 1, 0, S, Dh, S, bh, P, S, (H * S * S, S * S), h, E, (S * E, Dh), outb, 1, 3 * E,
         (S * 3 * E, Dh), nnt.make_epilogue(causal=3), 0.5),
        ("att_dq", 0, 0, S, Dh, S, bh, P, S, (H * S * S, S * S), h, 3 * E, (S * 3 * E, Dh), outb, 1, 3 * E,
         (S * 3 * E, Dh), nnt.make_epilogue(causal=2), 0.5),
        ("att_dk", 1, 0, S, Dh, S, bh, P, S, (H * S * S, S * S), h, 3 * E, (S * 3 * E, Dh), outb, 1, 3 * E,
         (S * 3 * E, Dh), nnt.make_epilogue(causal=3), 0.5),
        ("proj_dw+db", 1, 0, E, F, T, None, h, E, None, g, F, None, outf, 0, F, None, None, 1.0),
        ("fc_dw+db", 1, 0, F, E, T, None, g, F, None, h, E, None, outf, 0, E, None, None, 1.0),
        ("qkv_dw", 1, 0, 3 * E, E, T, None, h, 3 * E, None, h, E, None, outf, 0, E, None, None, 1.0),
        ("qkv_dx", 0, 0, T, E, 3 * E, None, h, 3 * E, None, w, E, None, outf, 0, E, None, None, 1.0),
        ("square8192", 0, 1, 8192, 8192, 8192, None, big, 8192, None, big, 8192, None, outb, 1, 8192, None,
         None, 1.0),
    ]
    ws = torch.zeros(64 << 20, device="cuda", dtype=torch.uint8)  # split-K / stream-K workspace (zero: flags)
    total = 0.0
    print(f"{'gemm':14s} {'M':>6s} {'N':>6s} {'K':>6s} {'batch':>8s} {'us':>8s} {'TFLOP/s':>8s}")
    for (name, ta, tb, M, N, K, batch, A, lda, sa, Bm, ldb, sb, Cm, cdt, ldc, sc, epi, frac) in cases:
        if a.only and name not in a.only.split(","):
            continue
        beta = 1.0 if name.endswith("_dw") else 0.0
        if name.endswith("_dw"):
            epi = nnt.make_epilogue(workspace=ws)
        if name.endswith("_dw+db"):
            beta = 1.0
            epi = nnt.make_epilogue(workspace=ws, a_rowsum=rowsum)
        if batch is None and not a.no_ws:  # unbatched: the workspace a block passes (stream-K slots)
            if epi is None:
                epi = nnt.make_epilogue(workspace=ws)
            else:
                epi.workspace, epi.workspace_bytes = ws.data_ptr(), ws.numel()
        if name == "square8192" and T * F < 8192 * 8192:
            outb = torch.empty(8192 * 8192, **bf)
            Cm = outb

        def run():
            nnt.nnt_tile_gemm(ta, tb, M, N, K, batch, 1.0, A, 1, lda, sa, Bm, 1, ldb, sb, beta, Cm, cdt, ldc, sc,
                              None, epi)
        for _ in range(3):
            run()
        # back-to-back launches between the events so host-side launch cost (ctypes, tensor-map
        # encoding) overlaps device time instead of being counted as idle GPU time
        ts = []
        reps = 10
        for _ in range(max(1, a.iters // 4)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                run()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / reps)
        ts.sort()
        us = ts[len(ts) // 2]
        nb = (batch[0] * batch[1]) if batch else 1
        fl = 2.0 * M * N * K * nb * frac
        if name != "square8192":
            total += us
        print(f"{name:14s} {M:6d} {N:6d} {K:6d} {str(nb):>8s} {us:8.1f} {fl / us / 1e6:8.1f}")
    print(f"total per layer {total:.1f} us  -> x{L} layers = {total * L / 1e3:.2f} ms")


if __name__ == "__main__":
    main()

"""Per-GPU compute of one tensor-parallel block shard (nnt_block_tp_*) at
group sizes R = 1, 2, 4, 8 on one B200: the two forward and three backward stages of one
shard (heads H/R, FFN 4E/R, the shard that adds the biases), graph-replayed, without the
four SUM reductions per block (one GPU: they are reported as bytes, T*E fp32 each).

    python tools/tp_bench.py [--config wide] [--rs 1,2,4,8]

Prints one JSON line per R: ms per block step, the shard's model TFLOP/s (the block's
PaLM-convention FLOPs / R), the reduction bytes per block step, and the time those would
take at the NVLink-5 per-direction bandwidth with a ring all-reduce (2 (R-1)/R T E 4 bytes
per reduction on each GPU) -- a model, not a measurement."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import nnt_inputs  # noqa: E402
from paper_2504_13236_b200 import model, nnt, tp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="wide")
    ap.add_argument("--rs", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    _, E, H, S, B = bench.CONFIGS[a.config]
    T = B * S
    sc = model.StackConfig(L=1, E=E, H=H, S=S, B=B, dtype="bf16")
    cfg = sc.block_cfg()
    p = nnt_inputs.make_params(E, seed=5, init="gpt2")
    flops = bench.model_flops_per_step(1, E, S, T)
    for R in [int(r) for r in a.rs.split(",")]:
        sp = tp.tp_shard(p, H, R, 0)
        t = nnt.nnt_block_tp(H // R, 4 * E // R, 1)
        dv = {n: torch.as_tensor(v).cuda() for n, v in sp.items()}
        w16 = {n: v.bfloat16() for n, v in dv.items() if n.startswith("w_")}
        g = {n: torch.zeros_like(v) for n, v in dv.items()}
        P, G = nnt.nnt_block_params(), nnt.nnt_block_grads()
        for n in sp:
            setattr(P, n, (w16[n] if n in w16 else dv[n]).data_ptr())
            setattr(G, n, g[n].data_ptr())
        sb, kb = nnt.nnt_block_tp_workspace_size(cfg, t)
        saved = torch.empty(sb, device="cuda", dtype=torch.uint8)
        scratch = torch.zeros(kb, device="cuda", dtype=torch.uint8)
        x = torch.randn(B, S, E, device="cuda")
        dy = torch.randn(B, S, E, device="cuda") / T
        x1, y, dh, dx = (torch.empty_like(x) for _ in range(4))

        def step():
            for st in (0, 1):
                nnt.nnt_block_tp_fwd(cfg, t, P, st, x, x1, y if st else None, saved, scratch)
            for st in (0, 1, 2):
                nnt.nnt_block_tp_bwd(cfg, t, P, st, x, x1, saved, scratch, dy, dh, dx if st == 2 else None, G, 0)

        for _ in range(3):
            step()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            step()
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            gr.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        ms = ts[len(ts) // 2]
        red_bytes = 4 * T * E * 4  # four reductions of T x E fp32 per block step
        ring = 4 * 2 * (R - 1) / R * T * E * 4
        print(json.dumps({"config": a.config, "R": R, "heads": H // R, "ffn": 4 * E // R, "ms_compute": ms,
                          "shard_model_tflops": flops / R / (ms / 1e3) / 1e12,
                          "reduction_bytes_per_block_step": red_bytes,
                          "ring_allreduce_ms_at_900GBps_model": ring / 900e9 * 1e3}), flush=True)
        del saved, scratch, gr


if __name__ == "__main__":
    main()

"""Per-iteration pipeline timeline of the fused attention kernels (CTA 0), from
nnt_attention_trace (microseconds from the first event).  Forward: K load issued, S MMA issued, S
seen by the epilogue, P staged, P seen by the MMA issuer, O MMA issued.  Backward: stage loads
issued, dP MMA issued, dP seen by the epilogue, dA staged, dA seen by the MMA issuer, dK MMA issued.

    python tools/attn_trace.py [--config small]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import nnt_inputs  # noqa: E402
from paper_2504_13236_b200 import model, nnt  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="small")
    a = ap.parse_args()
    L, E, H, S, B = bench.CONFIGS[a.config]
    sc = model.StackConfig(L=1, E=E, H=H, S=S, B=B, dtype="bf16")
    st = model.BlockStack(sc, [nnt_inputs.make_params(E, seed=1, init="gpt2")])
    x = torch.from_numpy(nnt_inputs.make_x(E, S, 0, B)).cuda()
    r = torch.from_numpy(nnt_inputs.make_r(E, S, 0, B)).cuda()
    st.train_step(x, r)
    torch.cuda.synchronize()
    nnt.nnt_attention_trace(1)
    st.train_step(x, r)
    torch.cuda.synchronize()
    out = np.zeros(2 * 6 * 256, np.uint64)
    nnt.nnt_attention_trace(0, out)
    for which, names in ((0, ("k_load", "S_issue", "S_ready", "P_done", "P_seen", "O_issue")),
                         (1, ("ld_issue", "dP_issue", "dP_ready", "dA_done", "dA_seen", "dK_issue"))):
        tr = out.reshape(2, 6, 256)[which].astype(np.float64)
        n = int((tr[5] > 0).sum())
        v = tr[:, :n][tr[:, :n] > 0]
        if not n or not v.size:
            continue
        t0 = v.min()
        print(("forward" if which == 0 else "backward") + " (CTA 0)")
        print("iter " + " ".join(f"{x:>9s}" for x in names))
        for g in range(n):
            row = [(tr[e, g] - t0) / 1e3 if tr[e, g] > 0 else float("nan") for e in range(6)]
            print(f"{g:4d} " + " ".join(f"{v:9.2f}" for v in row))


if __name__ == "__main__":
    main()

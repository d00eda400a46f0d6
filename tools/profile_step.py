"""One steady-state training step of a config inside cudaProfilerStart/Stop, for
`ncu --profile-from-start off` (launch lists, --set full captures).

    python tools/profile_step.py [--config small] [--warmup 2]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import nnt_inputs  # noqa: E402
from paper_2504_13236_b200 import model, nnt  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="small")
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--model", default=None, choices=["gpt2", "blocks"])
    ap.add_argument("--trace", default=None, help="write the step's launch-scope trace (class, kernels) here")
    a = ap.parse_args()
    L, E, H, S, B = bench.CONFIGS[a.config]
    L = a.layers or L
    mdl = a.model or bench.default_model(a.config)
    sc = model.StackConfig(L=L, E=E, H=H, S=S, B=B, dtype="bf16")
    layers = [nnt_inputs.make_params(E, seed=1234, layer=l, init="gpt2", n_layers=L) for l in range(L)]
    if mdl == "gpt2":
        V = bench.VOCAB
        st = model.GPT2Model(sc, V, layers, nnt_inputs.make_shell_params(V, S, E, seed=1234, init="gpt2"))
        tok = torch.from_numpy(nnt_inputs.make_ids(V, S, 0, B)).cuda()
        batch = (tok[:, :S].contiguous(), tok[:, 1:].contiguous())
    else:
        st = model.BlockStack(sc, layers)
        batch = (torch.from_numpy(nnt_inputs.make_x(E, S, 0, B)).cuda(),
                 torch.from_numpy(nnt_inputs.make_r(E, S, 0, B)).cuda())
    x, r = batch
    for _ in range(a.warmup):
        st.train_step(x, r)
    torch.cuda.synchronize()
    if a.trace:
        nnt.nnt_timing_enable(True)
    torch.cuda.cudart().cudaProfilerStart()
    st.train_step(x, r)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    if a.trace:
        with open(a.trace, "w") as f:
            json.dump(nnt.nnt_timing_trace(), f)
        nnt.nnt_timing_enable(False)
    print("profiled one step; loss", st.loss.item())


if __name__ == "__main__":
    main()

"""Device / host memory per GPT-2 layer and the largest trainable depth on one GPU, resident vs
with the host offloads of SURVEY §8(f) f4 (tiles that do not fit the
GPU live in host RAM).  Sizes come from the library (nnt_block_workspace_size) and the model's
flat layouts; CPU-only.

    python tools/capacity.py [--config xl] [--hbm-gb 180] [--host-gb 2000]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2504_13236_b200 import model, nnt  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="xl")
    ap.add_argument("--hbm-gb", type=float, default=180.0)
    ap.add_argument("--host-gb", type=float, default=2000.0)
    a = ap.parse_args()
    L, E, H, S, B = bench.CONFIGS[a.config]
    V, T = bench.VOCAB, B * S
    sc = model.StackConfig(L=L, E=E, H=H, S=S, B=B)
    saved, scratch = nnt.nnt_block_workspace_size(sc.block_cfg())
    _, _, n_layer = model.flat_layout(1, E)
    _, _, n_shell = model.shell_layout(V, S, E)
    x_layer = 4 * T * E                                  # the layer's fp32 input (resident)
    p_full, p_off = 18, 10                               # bytes/param: w, g, m, v fp32 + bf16 shadow; m, v on host
    fixed = scratch + n_shell * p_full + T * (V + 8) * 2 + 6 * 4 * T * E  # scratch, shell, logits, dy / dx / hf
    hbm = a.hbm_gb * 1e9
    rows = {}
    for name, act, opt in (("resident", False, False), ("act_offload", True, False), ("act+opt_offload", True, True)):
        dev_layer = x_layer + n_layer * (p_off if opt else p_full) + (0 if act else saved)
        dev_fixed = fixed + (2 * saved if act else 0) + (n_shell * (p_off - p_full) if opt else 0)
        host_layer = (saved if act else 0) + (n_layer * 8 if opt else 0)
        l_dev = int((hbm - dev_fixed) // dev_layer)
        l_host = int(a.host_gb * 1e9 // host_layer) if host_layer else None
        rows[name] = {"device_bytes_per_layer": dev_layer, "host_bytes_per_layer": host_layer,
                      "device_fixed_bytes": dev_fixed, "max_layers_device": l_dev, "max_layers_host_ram": l_host,
                      "max_layers": min(l_dev, l_host) if l_host else l_dev,
                      "pcie_bytes_per_layer_per_step": 2 * host_layer}
    print(json.dumps({"config": a.config, "E": E, "H": H, "S": S, "B": B, "saved_bytes_per_layer": saved,
                      "params_per_layer": n_layer, "hbm_gb": a.hbm_gb, "host_gb": a.host_gb, "modes": rows},
                     indent=1))


if __name__ == "__main__":
    main()

"""Times nnt_cross_entropy on the GPT-2 head's logits (T=8192 x V=50257 bf16, in place) and
checks the staged kernel against the re-reading one.  NNT_CE_RESTREAM=1 selects the latter.
    python tools/ce_bench.py            (prints us/launch and GB/s of 2 x T x V x 2 bytes)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2504_13236_b200 import nnt  # noqa: E402

T, V = 8192, 50257
Vp = -(-V // 8) * 8
g = torch.Generator(device="cuda").manual_seed(3)
src = (3.0 * torch.randn(T, Vp, device="cuda", generator=g)).to(torch.bfloat16)
lab = torch.randint(0, V, (T,), device="cuda", generator=g, dtype=torch.int32)
loss = torch.empty(T, device="cuda")
x = src.clone()
reps = 20
bufs = [src.clone() for _ in range(2)]  # 2 x 823 MB: the next launch's row is never L2-resident
fn = lambda b: nnt.nnt_cross_entropy(b, nnt.NNT_BF16, T, V, Vp, lab, 1.0 / T, loss, None, b, Vp)  # noqa: E731
fn(bufs[0])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(reps):
    fn(bufs[i % 2])
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / reps
print(f"cross_entropy {'restream' if os.environ.get('NNT_CE_RESTREAM') == '1' else 'staged'}: {us:.1f} us/launch, "
      f"{2.0 * T * V * 2 / us / 1e3:.0f} GB/s algorithmic (read + write of the logits)")
# one clean launch for the loss / gradient checksum (compared across variants by the caller)
fn(x)
torch.cuda.synchronize()
print(f"loss_sum {loss.double().sum().item():.9e} grad_sum {x[:, :V].double().abs().sum().item():.9e}")

import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import nnt_inputs
from gpu_util import dev, host
from paper_2504_13236_b200 import nnt
def run(M, N, K, ta, tb):
    a = nnt_inputs.make_matrix((K, M) if ta else (M, K), seed=M + N + 1, kind="int")
    b = nnt_inputs.make_matrix((N, K) if tb else (K, N), seed=M + 2 * N, kind="int")
    A, B = dev(a, torch.bfloat16), dev(b, torch.bfloat16)
    C = torch.zeros(M, N, device="cuda")
    nnt.nnt_tile_gemm(ta, tb, M, N, K, None, 1.0, A, 1, a.shape[1], None, B, 1, b.shape[1], None, 0.0, C, 0, N, None, None, None)
    torch.cuda.synchronize()
    want = (a.T if ta else a).astype(np.float64) @ (b.T if tb else b).astype(np.float64)
    got = host(C); bad = np.argwhere(got != want)
    msg = f"M={M} N={N} K={K} ta={ta} tb={tb}: bad={len(bad)}"
    if len(bad):
        r, c = bad[:, 0], bad[:, 1]
        msg += f" rows[{r.min()}..{r.max()}] cols[{c.min()}..{c.max()}] first={bad[:3].tolist()} got={got[tuple(bad[0])]} want={want[tuple(bad[0])]}"
    print(msg, flush=True)
for (M, N, K) in [(296, 200, 136), (296, 200, 128), (320, 200, 128), (296, 256, 128), (384, 200, 136), (512, 200, 136), (256, 200, 136), (264, 128, 64)]:
    for ta, tb in [(1, 0), (0, 0), (1, 1), (0, 1)]:
        run(M, N, K, ta, tb)

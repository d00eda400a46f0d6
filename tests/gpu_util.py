"""Helpers for the -m gpu parity tests (test infrastructure)."""
import json
import os

import numpy as np
import torch


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def rel_max(a, b):
    """max_i |a_i - b_i| / max_i |b_i| (SURVEY §8(c)'s element-wise parity metric)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def close(got, want, tol, what="", max_tol=None):
    """Parity assertion used by every block / shape / GPT-2 / kernel test (reading R32):
    the norm-wise error ||got - want||_2 / ||want||_2 < tol AND the element-wise error
    max|got - want| / max|want| < max_tol (default: the same bound).  The norm alone would let one
    wrong row, head or boundary tile of a large tensor pass; the element-wise bound does not.

    With NNT_PARITY_LOG=<file> every comparison is appended there as one JSON line (the evidence
    the bounds were chosen from)."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    assert got.shape == want.shape or got.size == want.size, (what, got.shape, want.shape)
    got = got.reshape(want.shape)
    assert np.all(np.isfinite(got)), f"{what}: non-finite values"
    r, m = rel(got, want), rel_max(got, want)
    max_tol = tol if max_tol is None else max_tol
    log = os.environ.get("NNT_PARITY_LOG")
    if log:
        import inspect
        test = os.environ.get("PYTEST_CURRENT_TEST", "").split(" ")[0]
        caller = inspect.stack()[1]
        with open(log, "a") as f:
            f.write(json.dumps({"test": test, "line": caller.lineno, "what": str(what), "n": int(want.size),
                                "rel": r, "rel_max": m, "tol": tol, "max_tol": max_tol}) + "\n")
    assert r < tol, f"{what}: norm-wise rel {r:.3e} >= {tol:.1e}"
    if not m < max_tol:
        i = int(np.abs(got - want).argmax())
        raise AssertionError(f"{what}: element-wise max rel {m:.3e} >= {max_tol:.1e} at flat index {i}: "
                             f"got {got.ravel()[i]:.6e} want {want.ravel()[i]:.6e} (max|want| "
                             f"{np.abs(want).max():.6e})")
    return r, m


def close_update(got_delta, want_delta, w_ref, rms_g, tol, what="", elementwise=True):
    """Parity of an Adam parameter update Δw = w_new - w_old (reading R32).

    Norm-wise over every element: ||Δ - Δref|| / ||Δref|| < tol.  Element-wise only where the
    update is well conditioned, i.e. where the gradient history is not small: Adam's step
    lr*m̂/(sqrt(v̂)+eps) normalises by the RMS gradient r = sqrt(v̂), so a gradient error δg moves
    an element's update by ~lr*δg/r (and at step 1 by lr*eps*δg/|g|^2 -- unbounded as |g| -> 0).
    With the fp32 path's gradient errors up to ~1e-6 of the tensor's largest gradient, an element
    whose RMS gradient rms_g (= sqrt(v) of the oracle's Adam state, or |g| for one step) is a
    fraction f of the tensor's largest moves by up to ~1e-6/f of lr: elements with f < 0.1 are left
    to the norm-wise bound (the update error of the rest is then <= ~1e-5 lr, well inside tol); the
    element-wise bound adds the fp32 storage rounding of w_new, 2^-23 * max|w| / max|Δref|.

    elementwise=False (multi-step trajectories): norm-wise only.  After one Adam step every element
    whose gradient is at rounding-noise level (exactly the key bias, R22) has moved by +-lr with a
    sign set by that noise, in either implementation, so two trajectories' parameters differ by
    O(lr) there and later updates cannot agree element by element; each step's gradients are
    compared element-wise at the GPU's own parameters instead (test_gpu_parity_full)."""
    got = np.asarray(got_delta, np.float64).ravel()
    want = np.asarray(want_delta, np.float64).ravel()
    rms = np.abs(np.asarray(rms_g, np.float64)).ravel()
    close(got, want, tol, what, max_tol=np.inf)
    if not elementwise:
        return
    keep = rms >= 0.1 * rms.max() if rms.size else rms.astype(bool)
    if not keep.any():
        return
    storage = 2.0 ** -23 * np.abs(np.asarray(w_ref, np.float64)).max() / max(np.abs(want).max(), 1e-300)
    close(got[keep], want[keep], np.inf, f"{what} (well-conditioned elements)", max_tol=tol + storage)


def dev(a, dtype=torch.float32):
    return torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


def host(t):
    return t.detach().float().cpu().numpy().astype(np.float64)


def bf16_round(a):
    """Round-to-nearest-even to bf16 and back (the value a bf16 tensor holds)."""
    return torch.as_tensor(np.asarray(a, np.float32)).bfloat16().float().numpy().astype(np.float64)

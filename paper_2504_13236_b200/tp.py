"""Tensor parallelism over the embedding-dimension tiles (PAPER.md:129-130:
"split entire data into tiles across embedding dimension"; reading R31 in DESIGN.md).

A group of R GPUs shares every block.  Rank r owns the tiles of the inner dimensions:
heads [r H/R, (r+1) H/R) (their q/k/v rows of W_qkv and columns of W_o) and hidden units
[r F/R, (r+1) F/R) (rows of W_fc, columns of W_pr); LayerNorm parameters and the two output
biases are replicated.  The activations along E are replicated; each block needs four SUM
reductions over the group (x1 and y in the forward, dL/dh2 and dL/dh1 in the backward),
issued between the stages of nnt_block_tp_fwd / nnt_block_tp_bwd.  Gradients of the
replicated parameters come out identical on every rank, so a plain per-rank Adam keeps the
replicas equal and no gradient all-reduce is needed (data parallelism would add one over a
second group).

Host logic only: the shard slicing (tp_shard / tp_unshard), the flat per-rank parameter
buffers and the collective schedule; every arithmetic step runs in libnnt.
"""
import math

import numpy as np
import torch

from . import nnt
from .model import ALIGN, StackConfig


def shard_shapes(E, H, R):
    """Shapes of one rank's block parameters (nnt.h, nnt_block_tp)."""
    assert H % R == 0 and (4 * E) % R == 0, (E, H, R)
    Ea, Fl = (H // R) * (E // H), 4 * E // R
    return {"ln1_g": (E,), "ln1_b": (E,), "w_qkv": (3 * Ea, E), "b_qkv": (3 * Ea,), "w_o": (E, Ea), "b_o": (E,),
            "ln2_g": (E,), "ln2_b": (E,), "w_fc": (Fl, E), "b_fc": (Fl,), "w_pr": (E, Fl), "b_pr": (E,)}


def _qkv_rows(E, H, R, r):
    Dh, hl = E // H, H // R
    a, b = r * hl * Dh, (r + 1) * hl * Dh
    return np.concatenate([np.arange(a, b), E + np.arange(a, b), 2 * E + np.arange(a, b)])


def tp_shard(p, H, R, r):
    """Rank r's slice of one block's full parameters (dict name -> array, GPT-2 layout:
    W_qkv [3E, E] q/k/v row blocks, head-major inside each)."""
    E = p["ln1_g"].shape[0]
    Dh, hl, Fl = E // H, H // R, 4 * E // R
    rows = _qkv_rows(E, H, R, r)
    a, b = r * hl * Dh, (r + 1) * hl * Dh
    f0, f1 = r * Fl, (r + 1) * Fl
    out = {n: p[n] for n in ("ln1_g", "ln1_b", "b_o", "ln2_g", "ln2_b", "b_pr")}
    out["w_qkv"], out["b_qkv"] = p["w_qkv"][rows], p["b_qkv"][rows]
    out["w_o"] = p["w_o"][:, a:b]
    out["w_fc"], out["b_fc"] = p["w_fc"][f0:f1], p["b_fc"][f0:f1]
    out["w_pr"] = p["w_pr"][:, f0:f1]
    return {n: np.ascontiguousarray(v) for n, v in out.items()}


def tp_unshard(shards, H):
    """Inverse of tp_shard over all R ranks (replicated parameters taken from rank 0)."""
    R = len(shards)
    E = shards[0]["ln1_g"].shape[0]
    full = {n: np.array(shards[0][n]) for n in ("ln1_g", "ln1_b", "b_o", "ln2_g", "ln2_b", "b_pr")}
    full["w_qkv"] = np.zeros((3 * E, E), dtype=shards[0]["w_qkv"].dtype)
    full["b_qkv"] = np.zeros(3 * E, dtype=shards[0]["b_qkv"].dtype)
    Dh, hl = E // H, H // R
    for r, s in enumerate(shards):
        rows = _qkv_rows(E, H, R, r)
        full["w_qkv"][rows], full["b_qkv"][rows] = s["w_qkv"], s["b_qkv"]
    full["w_o"] = np.concatenate([s["w_o"] for s in shards], axis=1)
    full["w_fc"] = np.concatenate([s["w_fc"] for s in shards], axis=0)
    full["b_fc"] = np.concatenate([s["b_fc"] for s in shards], axis=0)
    full["w_pr"] = np.concatenate([s["w_pr"] for s in shards], axis=1)
    assert full["w_o"].shape == (E, hl * Dh * R)
    return full


class TPBlockStack:
    """L blocks, each split over the process group's R ranks (one process per GPU; the group
    may be world size 1).  forward / probe_loss / backward / adam / train_step like
    model.BlockStack; params_of / grads_of give this rank's shard."""

    def __init__(self, cfg: StackConfig, layer_params, process_group, device="cuda", fused=False):
        """fused: the four SUMs per block run over peer memory (R35): the partial-producing GEMMs
        scatter their rows into the owners' receive slots, the owners reduce in rank order and
        gather the sums to every rank (libnnt nnt_tp_*); x1 / y / dh and the receive and flag
        buffers are then symmetric allocations (torch symmetric memory when R > 1, so every
        rank can address every other rank's copy).  Else NCCL all-reduces between the stages."""
        assert len(layer_params) == cfg.L and process_group is not None
        self.cfg, self.pg = cfg, process_group
        self.dev = torch.device(device)
        self.R = torch.distributed.get_world_size(process_group)
        self.rank = torch.distributed.get_rank(process_group)
        E, H, R = cfg.E, cfg.H, self.R
        self.shapes = shard_shapes(E, H, R)
        self.bcfg = cfg.block_cfg()
        self.tp = nnt.nnt_block_tp(H // R, 4 * E // R, 1 if self.rank == 0 else 0)
        # flat per-rank buffers (ALIGN-padded tensors, layer-major)
        self.offsets, off = [], 0
        for _ in range(cfg.L):
            d = {}
            for n, sh in self.shapes.items():
                k = math.prod(sh)
                d[n] = (off, k)
                off += -(-k // ALIGN) * ALIGN
            self.offsets.append(d)
        self.numel = off
        f32 = dict(device=self.dev, dtype=torch.float32)
        self.w, self.g, self.m, self.v = (torch.zeros(off, **f32) for _ in range(4))
        self.bf16 = cfg.dtype == "bf16"
        for l, P in enumerate(layer_params):
            sp = tp_shard({n: np.asarray(v, dtype=np.float32) for n, v in P.items()}, H, R, self.rank)
            for n, (o, k) in self.offsets[l].items():
                self.w[o:o + k].copy_(torch.as_tensor(sp[n]).reshape(-1).to(self.dev))
        self.w16 = torch.zeros(off, device=self.dev, dtype=torch.bfloat16) if self.bf16 else None
        if self.bf16:
            nnt.nnt_convert(self.w, nnt.NNT_F32, self.w16, nnt.NNT_BF16, off)
        self._params = [self._make_params(l) for l in range(cfg.L)]
        self._grads = [self._make_grads(l) for l in range(cfg.L)]
        saved_b, scratch_b = nnt.nnt_block_tp_workspace_size(self.bcfg, self.tp)
        self.saved = [torch.empty(saved_b, device=self.dev, dtype=torch.uint8) for _ in range(cfg.L)]
        self.scratch = torch.zeros(scratch_b, device=self.dev, dtype=torch.uint8)  # zero: split-K counters
        act = dict(device=self.dev, dtype=torch.float32)
        self.fused = fused
        self.peer = {}  # data_ptr of a symmetric buffer -> [rank q's address of it]
        if fused:
            T = cfg.B * cfg.S
            shape = (cfg.B, cfg.S, E)
            self.xs = [torch.empty(*shape, **act)] + [self._sym(shape, torch.float32) for _ in range(cfg.L)]
            self.x1 = [self._sym(shape, torch.float32) for _ in range(cfg.L)]
            self.dh = self._sym(shape, torch.float32)
            self.recv = self._sym((self.R, -(-T // self.R), E), torch.float32)
            self.flags = self._sym((2 * nnt.NNT_TP_MAX,), torch.int32)
            self.comm = nnt.make_tp_comm(self.R, self.rank, T, E, self.peer[self.recv.data_ptr()],
                                         self.peer[self.flags.data_ptr()])
            self.tp.comm = nnt.C.pointer(self.comm)
            self.epoch = 0
        else:
            self.xs = [torch.empty(cfg.B, cfg.S, E, **act) for _ in range(cfg.L + 1)]
            self.x1 = [torch.empty(cfg.B, cfg.S, E, **act) for _ in range(cfg.L)]
            self.dh = torch.empty(cfg.B, cfg.S, E, **act)
        self.dy = [torch.empty(cfg.B, cfg.S, E, **act) for _ in range(2)]
        self.loss = torch.zeros(1, **act)
        self.dot_scratch = torch.empty(nnt.nnt_dot_scratch_bytes(cfg.T * E), device=self.dev, dtype=torch.uint8)
        self.step_count = 0

    def view(self, buf, l, name):
        o, k = self.offsets[l][name]
        return buf[o:o + k]

    def _make_params(self, l):
        wsrc = self.w16 if self.bf16 else self.w
        p = nnt.nnt_block_params()
        for n in ("ln1_g", "ln1_b", "b_qkv", "b_o", "ln2_g", "ln2_b", "b_fc", "b_pr"):
            setattr(p, n, self.view(self.w, l, n).data_ptr())
        for n in ("w_qkv", "w_o", "w_fc", "w_pr"):
            setattr(p, n, self.view(wsrc, l, n).data_ptr())
        return p

    def _make_grads(self, l):
        gr = nnt.nnt_block_grads()
        for n in self.shapes:
            setattr(gr, n, self.view(self.g, l, n).data_ptr())
        return gr

    def params_of(self, l, buf=None):
        buf = self.w if buf is None else buf
        return {n: self.view(buf, l, n).reshape(sh) for n, sh in self.shapes.items()}

    def grads_of(self, l):
        return self.params_of(l, self.g)

    def _sym(self, shape, dtype):
        """A zeroed buffer that every rank of the group can address (self.peer[ptr][q] = rank q's
        copy as mapped here): a plain allocation when R == 1, torch symmetric memory otherwise."""
        if self.R == 1:
            t = torch.zeros(shape, device=self.dev, dtype=dtype)
            self.peer[t.data_ptr()] = [t.data_ptr()]
            return t
        import torch.distributed._symmetric_memory as symm_mem
        t = symm_mem.empty(shape, device=self.dev, dtype=dtype)
        t.zero_()
        h = symm_mem.rendezvous(t, self.pg)
        self.peer[t.data_ptr()] = [int(p) for p in h.buffer_ptrs]
        torch.distributed.barrier(group=self.pg)  # every rank's copy zeroed before any peer writes
        return t

    def _sum(self, t):
        if not self.fused:
            torch.distributed.all_reduce(t, group=self.pg)
            return
        # R35: the GEMMs have scattered this rank's partials; complete the SUM into every rank's t
        self.epoch += 1
        nnt.nnt_tp_signal(self.comm, self.epoch, 0)
        nnt.nnt_tp_reduce_gather(self.comm, self.peer[t.data_ptr()], self.epoch)
        nnt.nnt_tp_signal(self.comm, self.epoch, 1)
        nnt.nnt_tp_wait(self.comm, self.epoch)

    def forward(self, x=None):
        if x is not None:
            self.xs[0].copy_(x)
        for l in range(self.cfg.L):
            nnt.nnt_block_tp_fwd(self.bcfg, self.tp, self._params[l], 0, self.xs[l], self.x1[l], None, self.saved[l],
                                 self.scratch)
            self._sum(self.x1[l])
            nnt.nnt_block_tp_fwd(self.bcfg, self.tp, self._params[l], 1, self.xs[l], self.x1[l], self.xs[l + 1],
                                 self.saved[l], self.scratch)
            self._sum(self.xs[l + 1])
        return self.xs[-1]

    def probe_loss(self, r):
        """L = (1/T) sum <y, r>; dy = r / T (reading R13), on the replicated y."""
        n = self.cfg.T * self.cfg.E
        inv = 1.0 / self.cfg.T
        nnt.nnt_dot(self.xs[-1], r, n, inv, self.loss, self.dot_scratch, self.dot_scratch.numel())
        nnt.nnt_scale(r, inv, self.dy[0], n)
        return self.loss

    def backward(self):
        cur = 0
        for l in range(self.cfg.L - 1, -1, -1):
            args = (self.xs[l], self.x1[l], self.saved[l], self.scratch, self.dy[cur], self.dh)
            nnt.nnt_block_tp_bwd(self.bcfg, self.tp, self._params[l], 0, *args, None, self._grads[l], 0)
            self._sum(self.dh)
            nnt.nnt_block_tp_bwd(self.bcfg, self.tp, self._params[l], 1, *args, None, self._grads[l], 0)
            self._sum(self.dh)
            nnt.nnt_block_tp_bwd(self.bcfg, self.tp, self._params[l], 2, *args, self.dy[1 - cur], self._grads[l], 0)
            cur = 1 - cur
        return self.dy[cur]

    def adam(self):
        """Adam (or SGD) over this rank's shard; replicated parameters see identical gradients
        on every rank and stay bitwise equal."""
        self.step_count += 1
        c, t = self.cfg, self.step_count
        if c.optimizer == "sgd":
            nnt.nnt_sgd_step(self.numel, self.w, self.g, self.m, self.w16, c.lr, c.momentum, c.weight_decay)
            return
        hp = nnt.adam_hparams(c.lr, c.beta1, c.beta2, c.eps, c.weight_decay, t)
        nnt.nnt_adam_step(self.numel, self.w, self.g, self.m, self.v, self.w16, hp)

    def train_step(self, x=None, r=None):
        self.forward(x)
        self.probe_loss(r)
        self.backward()
        self.adam()
        return self.loss

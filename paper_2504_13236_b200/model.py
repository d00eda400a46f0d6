"""GPT-2 block stack driver: device memory, streams and process groups (torch)
around libnnt's C-ABI calls.  Every arithmetic step runs in libnnt kernels.

Memory layout (HBM, per GPU):
  * one flat fp32 master-parameter buffer, one flat fp32 gradient buffer, fp32
    Adam m and v, and a flat bf16 shadow of the parameters (GEMM operands on the
    bf16 path).  Layers are stored last-to-first and, inside a layer, in the
    order backward completes them ({proj}, {fc, ln2}, {out}, {qkv, ln1}), so the
    DP buckets (one per set) are contiguous slices in backward-completion order;
  * per layer: the input activation x_l (fp32 [B,S,E]) and the `saved`
    workspace of nnt_block_fwd; one `scratch` workspace shared by all layers.

Data parallelism (reading R14): batch tiles are partitioned
across ranks (nnt_partition), each rank runs the full stack on its tiles, and
gradient buckets are SUM-all-reduced with NCCL on a communication stream as
soon as nnt_block_bwd records the bucket's event, followed by Adam on that
bucket, overlapping the rest of the backward pass.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass

import torch

from . import nnt, offload

# (parameter, set) in flat-buffer order inside one layer
SETS = (("w_pr", "b_pr"), ("w_fc", "b_fc", "ln2_g", "ln2_b"), ("w_o", "b_o"), ("w_qkv", "b_qkv", "ln1_g", "ln1_b"))
ALIGN = 64  # elements; keeps every parameter view 256-byte aligned in fp32 and 128-byte in bf16


def param_shapes(E):
    F = 4 * E
    return {"ln1_g": (E,), "ln1_b": (E,), "w_qkv": (3 * E, E), "b_qkv": (3 * E,), "w_o": (E, E), "b_o": (E,),
            "ln2_g": (E,), "ln2_b": (E,), "w_fc": (F, E), "b_fc": (F,), "w_pr": (E, F), "b_pr": (E,)}


def flat_layout(L, E, shards=1):
    """Host bookkeeping of the flat parameter / gradient buffers (integer, bit-exact across ranks).

    Returns (offsets, buckets, numel): offsets[l][name] = (element offset, numel); buckets =
    [(layer, set index, begin, end)] in backward-completion order (layer L-1 first; inside a
    layer the SETS order), each bucket a contiguous slice; every tensor starts on an ALIGN
    boundary.  These buckets are the units of the DP all-reduce.
    shards > 1 (ZeRO-1): every bucket is two regions (`bucket_regions`), the
    set's GEMM weight and then its small parameters (biases, LayerNorm), each padded to a multiple
    of shards * ALIGN elements, so each splits into `shards` equal ALIGN-aligned owner slices:
    the weight region is all-gathered as bf16 shadows, the small one in fp32."""
    shapes = param_shapes(E)
    offsets = [None] * L
    buckets = []
    off = 0
    q = ALIGN * shards
    for l in range(L - 1, -1, -1):
        d = {}
        for si, names in enumerate(SETS):
            b0 = off
            for i, n in enumerate(names):
                numel = math.prod(shapes[n])
                d[n] = (off, numel)
                off += -(-numel // ALIGN) * ALIGN
                if shards > 1 and i == 0:  # end of the weight region
                    off = b0 + -(-(off - b0) // q) * q
            off = b0 + -(-(off - b0) // q) * q
            buckets.append((l, si, b0, off))
        offsets[l] = d
    return offsets, buckets, off


def bucket_regions(offsets, bucket, shards):
    """The ZeRO-1 gather regions of a flat_layout bucket (l, si, b0, b1): [(b0, mid, True), (mid,
    b1, False)] with [b0, mid) the set's GEMM weight (read by the kernels as a bf16 shadow on the
    bf16 path) and [mid, b1) its biases / LayerNorm parameters (read in fp32).  Unsharded, one
    region (b0, b1, True): its only owner updates the fp32 values of the whole bucket in place, so
    the bf16 shadows it writes are all the (identity) gather has to move."""
    l, si, b0, b1 = bucket
    if shards <= 1:
        return [(b0, b1, True)]
    mid = offsets[l][SETS[si][1]][0]
    return [(b0, mid, True), (mid, b1, False)]


def zero_shards(buckets, world, rank):
    """ZeRO-1 ownership (P:189-194 the update is per tile, so any partition of
    the flat range is legal): bucket [b0, b1) splits into `world` equal slices, rank r owns
    [b0 + r n, b0 + (r+1) n), n = (b1 - b0) / world.  Returns {b0: (s0, s1, c)}: the owned slice
    and its offset c in the rank's compact optimizer-state buffers (owned slices back to back).
    Integer bookkeeping, identical on every rank."""
    out, c = {}, 0
    for b in buckets:
        b0, b1 = b[-2], b[-1]
        assert (b1 - b0) % world == 0, (b0, b1, world)
        n = (b1 - b0) // world
        out[b0] = (b0 + rank * n, b0 + (rank + 1) * n, c)
        c += n
    return out, c


def zero1_bucket(g, w, b0, b1, s0, s1, group, update, w16=None):
    """One bucket (region) of the ZeRO-1 step: reduce-scatter the gradient slice
    so this rank holds the SUM over ranks of its owned part (in place: the owned part of g is the
    NCCL in-place receive position), update the owned parameters (update(s0, s1): Adam / SGD on
    the owned slice with the rank's compact state), all-gather the updated slices back into every
    rank's replica (in place again): the fp32 parameters w, or -- w16 given, a GEMM-weight region
    on the bf16 path -- only their bf16 shadows, which the update wrote for the owned slice (half
    the bytes; the fp32 master of a slice then lives on its owner alone, `BlockStack.gather_master`
    rebuilds the full vector off the step).  The caller's current stream orders it."""
    torch.distributed.reduce_scatter_tensor(g[s0:s1], g[b0:b1], group=group)
    update(s0, s1)
    if w16 is None:
        torch.distributed.all_gather_into_tensor(w[b0:b1], w[s0:s1], group=group)
    else:
        torch.distributed.all_gather_into_tensor(w16[b0:b1], w16[s0:s1], group=group)


def _update_kernel(o, b0, b1, m, v, t, stream, shadow):
    """The optimizer kernel on parameters [b0, b1) of owner o (BlockStack / GPT2Model) with the
    state views m, v (device memory: resident, or an offload staging slot)."""
    c, n = o.cfg, b1 - b0
    w16 = o.w16[b0:b1] if (o.bf16 and shadow) else None
    if c.optimizer == "sgd":  # the momentum buffer lives in m
        nnt.nnt_sgd_step(n, o.w[b0:b1], o.g[b0:b1], m, w16, c.lr, c.momentum, c.weight_decay, stream=stream)
        return
    nnt.nnt_adam_step(n, o.w[b0:b1], o.g[b0:b1], m, v, w16, o._hp(t), stream=stream)


def _distinct_stream(dev, avoid):
    """A torch stream that is none of `avoid` (torch's stream pool recycles its streams)."""
    taken = {s.cuda_stream for s in avoid if s is not None}
    for _ in range(128):
        s = torch.cuda.Stream(device=dev)
        if s.cuda_stream not in taken:
            return s
    raise RuntimeError("no distinct CUDA stream available")


class LossReader:
    """Pipelined device -> host reads of the per-step loss (what a training loop logs).

    push(loss) enqueues an asynchronous copy of this step's device loss into a pinned host slot
    and records an event on the current stream; pop() waits for the oldest pending copy and
    returns its value.  Reading step i's loss after step i+1 has been enqueued keeps the host
    from stalling the stream between steps; every step's loss is still read back."""

    def __init__(self, depth=2):
        self.buf = torch.empty(depth, dtype=torch.float32, pin_memory=True)
        self.ev = [torch.cuda.Event() for _ in range(depth)]
        self.pending = []
        self.n = 0

    def push(self, loss):
        if len(self.pending) == len(self.ev):
            raise RuntimeError("LossReader: pop() before pushing more than `depth` losses")
        slot = self.n % len(self.ev)
        self.n += 1
        self.buf[slot:slot + 1].copy_(loss.reshape(1).float(), non_blocking=True)
        self.ev[slot].record()
        self.pending.append(slot)

    def pop(self):
        slot = self.pending.pop(0)
        self.ev[slot].synchronize()
        return float(self.buf[slot])


@dataclass
class StackConfig:
    L: int
    E: int
    H: int
    S: int
    B: int                  # sequences on this GPU
    tile_e: int = 1024
    tile_f: int = 1024
    tile_s: int = 1024
    tile_t: int = 1024
    dtype: str = "bf16"     # "bf16" (tcgen05 path) or "f32" (SIMT fp32 path)
    ln_eps: float = 1e-5
    causal: bool = True
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.0
    optimizer: str = "adam"   # "adam" (Adam / AdamW with weight_decay) or "sgd" (SGD with momentum)
    momentum: float = 0.9     # SGD momentum
    # DP only: ZeRO-1 -- gradients reduce-scattered by bucket slice, optimizer
    # state for the owned slices only (1/world of m, v), updated parameters all-gathered
    zero: bool = False
    # optimizer state (Adam m, v / SGD momentum) in pinned host memory, streamed through device
    # staging slots by the copy engines around each update (offload.py)
    offload: bool = False
    # saved activations of the lowest `act_offload` layers in pinned host memory, moved by the copy
    # engines out after each forward and back before each backward (offload.HostActivations)
    act_offload: int = 0
    # weight/bias-gradient ops of the backward on a second stream (NNT_SIDE_STREAM=0 disables)
    side_stream: bool = os.environ.get("NNT_SIDE_STREAM", "1") != "0"
    # the side stream's join lagged by one layer (two scratch workspaces alternate between layers;
    # NNT_SIDE_LAG=1).  Off by default: measured no gain on the GPT-2 small / XL steps;
    # not combined with activation offload (a layer's saved slot is refilled right after its call)
    side_lag: bool = os.environ.get("NNT_SIDE_LAG", "0") == "1"
    # train_step without DP: each bucket's optimizer update runs on an update stream as soon as the
    # backward has finished with the bucket (its grad_ready event), overlapping the rest of the
    # backward -- the DP path's schedule without the all-reduce (NNT_OVERLAP_UPDATE=0 disables)
    overlap_update: bool = os.environ.get("NNT_OVERLAP_UPDATE", "1") != "0"

    def block_cfg(self):
        return nnt.nnt_block_cfg(self.E, self.H, self.S, self.B, self.tile_e, self.tile_f, self.tile_s, self.tile_t,
                                 nnt.NNT_BF16 if self.dtype == "bf16" else nnt.NNT_F32, self.ln_eps,
                                 1 if self.causal else 0)

    @property
    def T(self):
        return self.B * self.S


class BlockStack:
    def __init__(self, cfg: StackConfig, layer_params, device="cuda", process_group=None, global_tokens=None):
        """layer_params: list (len L) of dicts name -> host array/tensor (fp32)."""
        assert len(layer_params) == cfg.L
        self.cfg = cfg
        self.dev = torch.device(device)
        self.pg = process_group
        self.world = torch.distributed.get_world_size(process_group) if process_group is not None else 1
        # the DP path (bucketed all-reduce on a comm stream) runs whenever a process group is given,
        # also at world size 1 (so the GPU tests can exercise it on one device)
        self.dp = process_group is not None
        self.T_global = global_tokens if global_tokens is not None else cfg.T * self.world
        self.bcfg = cfg.block_cfg()
        E = cfg.E
        shapes = param_shapes(E)
        self.zero = cfg.zero and self.dp
        self.offsets, self.buckets, off = flat_layout(cfg.L, E, self.world if self.zero else 1)
        self.numel = off
        f32 = dict(device=self.dev, dtype=torch.float32)
        self.w = torch.zeros(off, **f32)
        self.g = torch.zeros(off, **f32)
        nstate = off
        if self.zero:
            self.regions = {b[2]: bucket_regions(self.offsets, b, self.world) for b in self.buckets}
            self.shards, nstate = zero_shards([r[:2] for b in self.buckets for r in self.regions[b[2]]], self.world,
                                              torch.distributed.get_rank(process_group))
        self.host_state = None
        if cfg.offload:
            self.host_state = offload.HostOptimizerState(nstate, self.dev, two_moments=cfg.optimizer != "sgd")
            self.m, self.v = self.host_state.m, self.host_state.v
        else:
            self.m = torch.zeros(nstate, **f32)
            self.v = torch.zeros(nstate, **f32)
        self.bf16 = cfg.dtype == "bf16"
        self.w16 = torch.zeros(off, device=self.dev, dtype=torch.bfloat16) if self.bf16 else None
        for l, P in enumerate(layer_params):
            for n, (o, k) in self.offsets[l].items():
                src = torch.as_tensor(P[n], dtype=torch.float32).reshape(-1)
                self.w[o:o + k].copy_(src.to(self.dev))
        if self.bf16:
            nnt.nnt_convert(self.w, nnt.NNT_F32, self.w16, nnt.NNT_BF16, off)
        self.step_count = 0
        # ---- views / ABI structs
        self._params = []
        self._grads = []
        for l in range(cfg.L):
            self._params.append(self._make_params(l))
            self._grads.append(self._make_grads(l))
        saved_b, scratch_b = nnt.nnt_block_workspace_size(self.bcfg)
        self.n_off = max(0, min(cfg.act_offload, cfg.L))
        self.act_host = offload.HostActivations(self.n_off, saved_b, self.dev) if self.n_off else None
        self.saved = [self.act_host.slot(l) if l < self.n_off else
                      torch.empty(saved_b, device=self.dev, dtype=torch.uint8) for l in range(cfg.L)]
        self.scratch = torch.zeros(scratch_b, device=self.dev, dtype=torch.uint8)  # zero: split-K counters
        act = dict(device=self.dev, dtype=torch.float32)
        self.xs = [torch.empty(cfg.B, cfg.S, E, **act) for _ in range(cfg.L + 1)]
        self.dy = [torch.empty(cfg.B, cfg.S, E, **act) for _ in range(2)]
        # links between consecutive blocks' backward passes (the LayerNorm backward kernels):
        # layer l's LayerNorm-1 backward also makes sum_t dx (layer l-1's projection-bias gradient)
        # and, on the bf16 path, the bf16 copy of dx that layer l-1's projection GEMMs read
        self.chain = True
        self.dy16 = ([torch.empty(cfg.B, cfg.S, E, device=self.dev, dtype=torch.bfloat16) for _ in range(2)]
                     if self.chain and cfg.dtype == "bf16" else None)
        self.loss = torch.zeros(1, **act)
        self.dot_scratch = torch.empty(nnt.nnt_dot_scratch_bytes(cfg.T * E), device=self.dev, dtype=torch.uint8)
        # every stream of this model distinct (torch's round-robin stream pool recycles streams);
        # cap_stream: graphs are captured on it (torch.cuda.graph would take one from the pool)
        used = [] if self.host_state is None else [self.host_state.h2d, self.host_state.d2h]
        if self.act_host is not None:
            used += [self.act_host.h2d, self.act_host.d2h]
        # bucketed: gradient buckets handed to the comm / update stream on their grad_ready events
        self.bucketed = self.dp or cfg.overlap_update
        self.comm = _distinct_stream(self.dev, used) if self.bucketed else None
        self.side = _distinct_stream(self.dev, used + [self.comm]) if cfg.side_stream else None
        self.cap_stream = _distinct_stream(self.dev, used + [self.comm, self.side])
        self.events = [[torch.cuda.Event() for _ in range(4)] for _ in range(cfg.L)] if self.bucketed else None
        # lagged side-stream join: layer l uses scratch l % 2 and records its side ops' completion in
        # ev_side[l % 2]; the main stream waits on it before layer l - 2 reuses that scratch, and
        # the layer below waits on it before overwriting the dy its side ops read
        self.lag = self.side is not None and cfg.side_lag and cfg.L > 1 and not self.n_off
        self.scratch2 = torch.zeros_like(self.scratch) if self.lag else None  # zero: split-K counters
        self.ev_side = [torch.cuda.Event(), torch.cuda.Event()] if self.lag else None
        created = (self.events or []) + ([self.ev_side] if self.lag else [])
        if created:  # torch creates the CUDA event handles lazily, at the first record()
            for evs in created:
                for e in evs:
                    e.record()
            torch.cuda.synchronize(self.dev)
        self._graph_hp = None  # during enable_graph()'s capture: Adam reads its bias corrections from the device

    # ------------------------------------------------------------ views
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
        for n in param_shapes(self.cfg.E):
            setattr(gr, n, self.view(self.g, l, n).data_ptr())
        return gr

    def params_of(self, l, buf=None):
        shapes = param_shapes(self.cfg.E)
        buf = self.w if buf is None else buf
        return {n: self.view(buf, l, n).reshape(shapes[n]) for n in shapes}

    def grads_of(self, l):
        return self.params_of(l, self.g)

    # ------------------------------------------------------------ passes
    def forward(self, x=None):
        if x is not None:
            self.xs[0].copy_(x)
        ah = self.act_host
        compute = torch.cuda.current_stream()
        if ah is not None:
            ah.begin(compute)
        for l in range(self.cfg.L):
            if ah is not None and l < self.n_off:
                ah.before_fwd(l, compute)
            nnt.nnt_block_fwd(self.bcfg, self._params[l], self.xs[l], self.xs[l + 1], self.saved[l], self.scratch)
            if ah is not None and l < self.n_off:
                ah.after_fwd(l, compute)
        return self.xs[-1]

    def probe_loss(self, r):
        """L = (1/T_global) sum <y, r> on device; dy = r / T_global (reading R13)."""
        n = self.cfg.T * self.cfg.E
        inv = 1.0 / self.T_global
        nnt.nnt_dot(self.xs[-1], r, n, inv, self.loss, self.dot_scratch, self.dot_scratch.numel())
        nnt.nnt_scale(r, inv, self.dy[0], n)
        return self.loss

    def backward(self, overlap_optimizer=None, top_done=False):
        """Backward through the stack.  With DP every gradient bucket is SUM-all-reduced on the comm
        stream as soon as it is complete; with overlap_optimizer (default: with DP) the bucket's
        optimizer update follows it there, overlapping the rest of the backward.  Without DP,
        overlap_optimizer=True runs the per-bucket updates the same way (no all-reduce).

        top_done: the caller already wrote sum_t dy into the top layer's b_pr gradient and (bf16)
        the bf16 copy of dy into self.dy16[0] (GPT2Model's final-LayerNorm backward does)."""
        cur = 0
        compute = torch.cuda.current_stream()
        if overlap_optimizer is None:
            overlap_optimizer = self.dp
        dp = self.dp or bool(overlap_optimizer)
        assert not dp or self.events is not None, "per-bucket updates need StackConfig.overlap_update or DP"
        ah = self.act_host
        lag = self.lag
        for l in range(self.cfg.L - 1, -1, -1):
            if ah is not None and l < self.n_off:
                ah.before_bwd(l, compute)
            ev = self.events[l] if dp else None
            links = None
            scratch = self.scratch
            if lag:
                scratch = self.scratch if l % 2 == 0 else self.scratch2
                if l <= self.cfg.L - 3:  # layer l + 2's side ops (same scratch) are done
                    compute.wait_event(self.ev_side[l % 2])
            if self.chain or lag:
                links = nnt.nnt_block_bwd_links()
            if lag:
                links.side_done = self.ev_side[l % 2].cuda_event
                links.wait_before_dx = self.ev_side[(l + 1) % 2].cuda_event if l < self.cfg.L - 1 else None
            if self.chain:
                done = l < self.cfg.L - 1 or top_done
                links.dy_colsum_done = 1 if done else 0
                links.dy_bf16 = self.dy16[cur].data_ptr() if (done and self.dy16 is not None) else None
                if l > 0:
                    links.dx_colsum = self.view(self.g, l - 1, "b_pr").data_ptr()
                    links.dx_bf16 = self.dy16[1 - cur].data_ptr() if self.dy16 is not None else None
            nnt.nnt_block_bwd_streams(self.bcfg, self._params[l], self.xs[l], self.saved[l], scratch,
                                      self.dy[cur], self.dy[1 - cur], self._grads[l], 0, ev,
                                      side_stream=self.side, links=links)
            if ah is not None and l < self.n_off:
                ah.after_bwd(l, compute)
                ah.prefetch(l - 2, after_bwd_of=l)  # slot l % 2 is free: bring back layer l - 2
            if dp:
                for si in range(4):
                    self._reduce_bucket(l, si, ev[si], overlap_optimizer)
            cur = 1 - cur
        if lag:  # the bottom layer's side ops (the last lagged ones) before anything that follows
            compute.wait_event(self.ev_side[0])
        if ah is not None:
            ah.join(compute)
        if dp:
            compute.wait_stream(self.comm)
        return self.dy[cur]

    def _bucket_range(self, l, si):
        for (bl, bs, b0, b1) in self.buckets:
            if bl == l and bs == si:
                return b0, b1
        raise KeyError((l, si))

    def _reduce_bucket(self, l, si, event, with_adam):
        b0, b1 = self._bucket_range(l, si)
        with torch.cuda.stream(self.comm):
            self.comm.wait_event(event)
            if self.zero:
                assert with_adam, "ZeRO-1 updates inside the bucket step"
                self._zero_bucket(b0, b1, self.step_count + 1)
                return
            if self.dp:
                torch.distributed.all_reduce(self.g[b0:b1], group=self.pg)
            if with_adam:
                self._adam_range(b0, b1, self.step_count + 1, stream=self.comm)

    def _zero_bucket(self, b0, b1, t):
        for r0, r1, is_w in self.regions[b0]:
            s0, s1, c = self.shards[r0]
            # bf16 path: the weight region's owner writes the bf16 shadows of its slice and only they
            # are gathered; the small parameters (read in fp32) are gathered in fp32
            shadow = self.bf16 and is_w
            zero1_bucket(self.g, self.w, r0, r1, s0, s1, self.pg,
                         lambda a, b, c=c, shadow=shadow: self._update(a, b, c, t, self.comm, shadow=shadow),
                         w16=self.w16 if shadow else None)

    def gather_master(self):
        """ZeRO-1 on the bf16 path keeps the fp32 master of each weight slice on its owner only
        (the step gathers the bf16 shadows): all-gather the fp32 weight regions so every replica's
        `w` is the full current parameter vector again (checkpoints, tests).  Off the step path;
        a no-op without ZeRO-1 or on the fp32 path."""
        if not (self.zero and self.bf16):
            return
        torch.cuda.current_stream().wait_stream(self.comm)
        for b in self.buckets:
            for r0, r1, is_w in self.regions[b[2]]:
                if is_w:
                    s0, s1, _ = self.shards[r0]
                    torch.distributed.all_gather_into_tensor(self.w[r0:r1], self.w[s0:s1], group=self.pg)

    def _hparams(self, t):
        c = self.cfg
        return nnt.adam_hparams(c.lr, c.beta1, c.beta2, c.eps, c.weight_decay, t)

    def _adam_range(self, b0, b1, t, stream=None):
        self._update(b0, b1, b0, t, stream, shadow=True)

    def _update(self, b0, b1, c0, t, stream, shadow):
        """Optimizer step on parameters [b0, b1) with state at [c0, c0 + b1 - b0) of m / v."""
        if self.host_state is not None:
            self.host_state.apply([(c0, c0 + b1 - b0)],
                                  lambda a, b, m, v: _update_kernel(self, b0 + a - c0, b0 + b - c0, m, v, t, stream,
                                                                    shadow), stream)
            return
        _update_kernel(self, b0, b1, self.m[c0:c0 + b1 - b0], self.v[c0:c0 + b1 - b0], t, stream, shadow)

    def _hp(self, t):
        return self._graph_hp if self._graph_hp is not None else self._hparams(t)

    def adam(self):
        """Adam over every parameter (one launch over the flat buffer); bias corrections in fp64 on host."""
        self.step_count += 1
        self._adam_range(0, self.numel, self.step_count)

    def train_step(self, x=None, r=None):
        """forward -> probe loss -> backward (+ DP all-reduce) -> Adam.  Returns the device loss tensor.

        x, r: [B,S,E] fp32, on this device or on the host (pinned host tensors are
        copied asynchronously into the device input buffers first).  After
        enable_graph() the whole step is one CUDA-graph replay."""
        if getattr(self, "graph", None) is not None:
            return self._graph_step(x, r)
        if x is not None and x.device.type == "cpu":
            self.xs[0].copy_(x, non_blocking=True)
            x = None
        if r is not None and r.device.type == "cpu":
            if not hasattr(self, "r_buf"):
                self.r_buf = torch.empty_like(self.xs[0])
            self.r_buf.copy_(r, non_blocking=True)
            r = self.r_buf
        self.forward(x)
        self.probe_loss(r)
        if self.bucketed:  # per-bucket all-reduce (DP) and update on the comm / update stream
            self.backward(overlap_optimizer=True)
            self.step_count += 1
        else:
            self.backward()
            self.adam()
        return self.loss

    # ------------------------------------------------------------ CUDA graph
    def enable_graph(self):
        """Capture one whole training step (Adam step counter advanced on the device, fp64
        bias corrections, then forward, probe loss, backward, Adam) as a CUDA graph; later
        train_step calls copy the batch into the static input buffers and replay it.  This
        removes the host cost of ~500 launches (ctypes + TMA-descriptor encoding) per step.

        With a process group (DP) the capture forks the communication stream off the compute
        stream at every bucket event: each bucket's NCCL all-reduce and Adam are graph nodes
        that overlap the rest of the backward pass, joined before the step ends."""
        self.graph = self.capture_graph()
        return self.graph

    def capture_graph(self):
        """One training step as a new CUDA graph (replay = one step; shares the step counter and
        input buffers with enable_graph's graph).  With nnt_timing_enable(True) around the capture
        the libnnt launch scopes become event-record nodes, timing every kernel class inside the
        replayed graph (bench.py's per-kernel roofline)."""
        dev = self.dev
        if not hasattr(self, "r_buf"):
            self.r_buf = torch.empty_like(self.xs[0])
        if not hasattr(self, "t_dev"):
            self.t_dev = torch.tensor([self.step_count], device=dev, dtype=torch.int64)
            self.bc_dev = torch.zeros(2, device=dev, dtype=torch.float32)
        c = self.cfg
        hp = nnt.adam_hparams(c.lr, c.beta1, c.beta2, c.eps, c.weight_decay)
        hp.bias_corr_dev = self.bc_dev.data_ptr()
        if self.dp:  # the communicator must exist before capture: one eager collective on the comm stream
            with torch.cuda.stream(self.comm):
                torch.distributed.all_reduce(torch.zeros(1, device=dev), group=self.pg)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        self._graph_hp = hp
        try:
            with torch.cuda.graph(g, stream=self.cap_stream):
                nnt.nnt_adam_tick(c.beta1, c.beta2, self.t_dev, self.bc_dev)
                self.forward()
                self.probe_loss(self.r_buf)
                if self.bucketed:
                    self.backward(overlap_optimizer=True)
                else:
                    self.backward()
                    self._adam_range(0, self.numel, 0)
        finally:
            self._graph_hp = None  # eager steps keep host-side bias corrections
        return g

    def _graph_step(self, x, r):
        if x is not None:
            self.xs[0].copy_(x, non_blocking=True)
        if r is not None:
            self.r_buf.copy_(r, non_blocking=True)
        self.graph.replay()
        self.step_count += 1
        return self.loss


# ---------------------------------------------------------------------------------------------
# Full GPT-2: embedding -> BlockStack -> final LayerNorm -> tied LM head ->
# cross-entropy.  All arithmetic in libnnt kernels (nnt_embedding_*, nnt_layernorm_*,
# nnt_tile_gemm for the two LM-head products, nnt_cross_entropy, nnt_dot, nnt_adam_step).
# ---------------------------------------------------------------------------------------------
SHELL = ("wte", "wpe", "lnf_g", "lnf_b")


def shell_layout(V, S_max, E, shards=1):
    """Flat layout of the shell parameters (ALIGN-padded; the total a multiple of shards * ALIGN
    for ZeRO-1): name -> (offset, numel), total."""
    shapes = {"wte": (V, E), "wpe": (S_max, E), "lnf_g": (E,), "lnf_b": (E,)}
    off, d = 0, {}
    for n in SHELL:
        k = math.prod(shapes[n])
        d[n] = (off, k)
        off += -(-k // ALIGN) * ALIGN
    q = ALIGN * shards
    return d, shapes, -(-off // q) * q


class GPT2Model:
    """GPT-2 with tied token embedding / LM head on one GPU's batch tiles (DP: a process group;
    the shell gradients are one more all-reduce bucket, issued after the embedding backward)."""

    def __init__(self, cfg: StackConfig, V, layer_params, shell_params, device="cuda", process_group=None,
                 global_tokens=None):
        self.cfg, self.V = cfg, V
        self.stack = BlockStack(cfg, layer_params, device, process_group, global_tokens)
        st = self.stack
        self.dev = st.dev
        E, T = cfg.E, cfg.T
        self.bf16 = cfg.dtype == "bf16"
        self.dt = nnt.NNT_BF16 if self.bf16 else nnt.NNT_F32
        tdt = torch.bfloat16 if self.bf16 else torch.float32
        self.S_max = shell_params["wpe"].shape[0]
        self.offsets, self.shapes, n = shell_layout(V, self.S_max, E, st.world if st.zero else 1)
        f32 = dict(device=self.dev, dtype=torch.float32)
        self.w, self.g = torch.zeros(n, **f32), torch.zeros(n, **f32)
        nstate = n
        if st.zero:  # the shell is one more bucket
            self.shard, nstate = zero_shards([(0, n)], st.world, torch.distributed.get_rank(st.pg))
            self.shard = self.shard[0]
        self.host_state = None
        if cfg.offload:
            self.host_state = offload.HostOptimizerState(nstate, self.dev, two_moments=cfg.optimizer != "sgd")
            self.m, self.v = self.host_state.m, self.host_state.v
        else:
            self.m, self.v = torch.zeros(nstate, **f32), torch.zeros(nstate, **f32)
        for name, (o, k) in self.offsets.items():
            self.w[o:o + k].copy_(torch.as_tensor(shell_params[name], dtype=torch.float32).reshape(-1).to(self.dev))
        self.numel = n
        self.w16 = torch.zeros(n, device=self.dev, dtype=torch.bfloat16) if self.bf16 else None
        if self.bf16:
            nnt.nnt_convert(self.w, nnt.NNT_F32, self.w16, nnt.NNT_BF16, n)
        self.Vp = -(-V // 8) * 8  # logits row pitch: 16-byte rows for TMA / vector access
        self.ids = torch.zeros(T, device=self.dev, dtype=torch.int32)
        self.labels = torch.zeros(T, device=self.dev, dtype=torch.int32)
        self.hf = torch.empty(T, E, device=self.dev, dtype=tdt)
        self.mean, self.rstd = torch.empty(T, **f32), torch.empty(T, **f32)
        self.logits = torch.empty(T, self.Vp, device=self.dev, dtype=tdt)
        self.loss_rows = torch.empty(T, **f32)
        self.ones = torch.ones(T, **f32)
        self.dhf = torch.empty(T, E, **f32)
        # split-K workspace of dh_f = dlogits wte (K = V: the library splits K when the tile grid
        # fills its last round badly); None when the library would not split
        wsb = nnt.nnt_tile_gemm_workspace_bytes(T, E, V, nnt.NNT_F32) if self.bf16 else 0
        self.dh_ws = torch.zeros(wsb, device=self.dev, dtype=torch.uint8) if wsb else None  # zero: counters
        self.dh_epi = nnt.make_epilogue(workspace=self.dh_ws) if wsb else None
        self.lnf_scr = torch.empty(nnt.nnt_layernorm_bwd_scratch_bytes(T, E), device=self.dev, dtype=torch.uint8)
        self.emb_scr = torch.empty(nnt.nnt_embedding_bwd_scratch_bytes(T, V), device=self.dev, dtype=torch.uint8)
        self.dot_scr = torch.empty(nnt.nnt_dot_scratch_bytes(T), device=self.dev, dtype=torch.uint8)
        self.loss = torch.zeros(1, **f32)
        self.step_count = 0
        self.ev_shell = torch.cuda.Event()
        if st.bucketed:
            self.ev_shell.record()
        self.graph = None

    def view(self, buf, name):
        o, k = self.offsets[name]
        return buf[o:o + k]

    def params(self):
        return {n: self.view(self.w, n).reshape(self.shapes[n]) for n in SHELL}

    def grads(self):
        return {n: self.view(self.g, n).reshape(self.shapes[n]) for n in SHELL}

    # ------------------------------------------------------------------ passes
    def forward(self, ids=None, labels=None):
        c, st = self.cfg, self.stack
        T, E, V = c.T, c.E, self.V
        if ids is not None:
            self.ids.copy_(ids.reshape(-1), non_blocking=True)
        if labels is not None:
            self.labels.copy_(labels.reshape(-1), non_blocking=True)
        nnt.nnt_embedding_fwd(self.ids, T, c.S, self.view(self.w, "wte"), V, self.view(self.w, "wpe"), E, st.xs[0])
        st.forward()
        nnt.nnt_layernorm_fwd(st.xs[-1], T, E, E, c.tile_e, self.view(self.w, "lnf_g"), self.view(self.w, "lnf_b"),
                              c.ln_eps, self.hf, self.dt, E, self.mean, self.rstd)
        wsrc = self.w16 if self.bf16 else self.w
        # logits = h_f wte^T (tied LM head), C in the compute dtype with a 16-byte row pitch
        nnt.nnt_tile_gemm(nnt.NNT_NOTRANS, nnt.NNT_TRANS, T, V, E, None, 1.0, self.hf, self.dt, E, None,
                          self.view(wsrc, "wte"), self.dt, E, None, 0.0, self.logits, self.dt, self.Vp, None,
                          (c.tile_t, c.tile_e, c.tile_e))
        # cross-entropy: per-token loss and, in place, dlogits = (softmax - onehot) / T_global
        inv = 1.0 / st.T_global
        nnt.nnt_cross_entropy(self.logits, self.dt, T, V, self.Vp, self.labels, inv, self.loss_rows, None,
                              self.logits, self.Vp)
        nnt.nnt_dot(self.loss_rows, self.ones, T, inv, self.loss, self.dot_scr, self.dot_scr.numel())
        return self.loss

    def backward(self, overlap_optimizer=None):
        """Backward through the whole model.  overlap_optimizer (default: with DP): every bucket's
        update -- the blocks' and, after the embedding backward, the shell's -- runs on the comm /
        update stream as soon as its gradients are complete (after their all-reduce with DP)."""
        c, st = self.cfg, self.stack
        if overlap_optimizer is None:
            overlap_optimizer = st.dp
        T, E, V = c.T, c.E, self.V
        wsrc = self.w16 if self.bf16 else self.w
        tiles = (c.tile_t, c.tile_e, c.tile_e)
        # dh_f = dlogits wte ; dwte = dlogits^T h_f (the LM-head half of the tied gradient)
        nnt.nnt_tile_gemm(nnt.NNT_NOTRANS, nnt.NNT_NOTRANS, T, E, V, None, 1.0, self.logits, self.dt, self.Vp, None,
                          self.view(wsrc, "wte"), self.dt, E, None, 0.0, self.dhf, nnt.NNT_F32, E, None, tiles,
                          self.dh_epi)
        nnt.nnt_tile_gemm(nnt.NNT_TRANS, nnt.NNT_NOTRANS, V, E, T, None, 1.0, self.logits, self.dt, self.Vp, None,
                          self.hf, self.dt, E, None, 0.0, self.view(self.g, "wte"), nnt.NNT_F32, E, None, tiles)
        top = st.chain  # the final LayerNorm's backward also makes the top block's b_pr sum and dy copy
        nnt.nnt_layernorm_bwd(self.dhf, E, st.xs[-1], E, self.mean, self.rstd, self.view(self.w, "lnf_g"), T, E,
                              None, st.dy[0], E, st.dy16[0] if (top and st.dy16 is not None) else None,
                              self.view(self.g, "lnf_g"), self.view(self.g, "lnf_b"),
                              st.view(st.g, c.L - 1, "b_pr") if top else None, 0,
                              self.lnf_scr, self.lnf_scr.numel())
        dx0 = st.backward(overlap_optimizer=overlap_optimizer, top_done=top)
        # dwte accumulates onto the LM head's half (written with beta = 0 above); dwpe has no other
        # producer and is overwritten
        nnt.nnt_embedding_bwd(self.ids, T, c.S, dx0, E, self.view(self.g, "wte"), V, self.view(self.g, "wpe"), 1, 0,
                              self.emb_scr, self.emb_scr.numel())
        if st.dp or overlap_optimizer:  # the shell bucket: all-reduce (DP) + update on the comm stream
            self.ev_shell.record()
            with torch.cuda.stream(st.comm):
                st.comm.wait_event(self.ev_shell)
                if not st.dp:
                    self._adam(st.step_count + 1, stream=st.comm)
                elif st.zero:
                    s0, s1, _ = self.shard
                    zero1_bucket(self.g, self.w, 0, self.numel, s0, s1, st.pg,
                                 lambda a, b: self._update(a, b, 0, st.step_count + 1, st.comm, shadow=False))
                    if self.bf16:
                        nnt.nnt_convert(self.w, nnt.NNT_F32, self.w16, nnt.NNT_BF16, self.numel, stream=st.comm)
                else:
                    torch.distributed.all_reduce(self.g, group=st.pg)
                    self._adam(st.step_count + 1, stream=st.comm)
            torch.cuda.current_stream().wait_stream(st.comm)
        return dx0

    def _adam(self, t, stream=None):
        self._update(0, self.numel, 0, t, stream, shadow=True)

    def _hp(self, t):
        return self.stack._hp(t)

    _update = BlockStack._update

    def adam(self):
        self.stack.adam()
        self.step_count = self.stack.step_count
        self._adam(self.step_count)

    def gather_master(self):
        """The block stack's fp32 masters after ZeRO-1 bf16 steps (BlockStack.gather_master); the
        shell bucket is gathered in fp32 every step (the embedding forward reads fp32 tables)."""
        self.stack.gather_master()

    def train_step(self, ids=None, labels=None):
        """forward -> cross-entropy -> backward (+ DP all-reduce) -> Adam; returns the device loss."""
        if self.graph is not None:
            if ids is not None:
                self.ids.copy_(ids.reshape(-1), non_blocking=True)
            if labels is not None:
                self.labels.copy_(labels.reshape(-1), non_blocking=True)
            self.graph.replay()
            self.stack.step_count += 1
            self.step_count = self.stack.step_count
            return self.loss
        self.forward(ids, labels)
        if self.stack.bucketed:
            self.backward(overlap_optimizer=True)
            self.stack.step_count += 1
            self.step_count = self.stack.step_count
        else:
            self.backward()
            self.adam()
        return self.loss

    def capture_graph(self):
        """One training step as a CUDA graph (see BlockStack.capture_graph)."""
        st, c = self.stack, self.cfg
        dev = self.dev
        if not hasattr(st, "t_dev"):
            st.t_dev = torch.tensor([st.step_count], device=dev, dtype=torch.int64)
            st.bc_dev = torch.zeros(2, device=dev, dtype=torch.float32)
        hp = nnt.adam_hparams(c.lr, c.beta1, c.beta2, c.eps, c.weight_decay)
        hp.bias_corr_dev = st.bc_dev.data_ptr()
        if st.dp:
            with torch.cuda.stream(st.comm):
                torch.distributed.all_reduce(torch.zeros(1, device=dev), group=st.pg)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        st._graph_hp = hp
        try:
            with torch.cuda.graph(g, stream=st.cap_stream):
                nnt.nnt_adam_tick(c.beta1, c.beta2, st.t_dev, st.bc_dev)
                self.forward()
                if st.bucketed:
                    self.backward(overlap_optimizer=True)
                else:
                    self.backward()
                    st._adam_range(0, st.numel, 0)
                    self._adam(0)
        finally:
            st._graph_hp = None
        return g

    def enable_graph(self):
        self.graph = self.capture_graph()
        return self.graph

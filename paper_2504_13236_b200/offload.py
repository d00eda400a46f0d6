"""Optimizer state resident in pinned host memory (PAPER.md:91-98, 204-205:
tiles that do not fit in GPU memory live in host RAM and are moved by the runtime).

The Adam moments (or the SGD momentum) of a parameter range stay in page-locked host RAM.
An update streams them through two device staging slots in chunks: the copy engine
brings chunk i+1 in (host-to-device stream) while the update kernel works on chunk i (the
caller's stream) and chunk i-1 is written back (device-to-host stream).  Device memory for
the state drops from 8 bytes per parameter to 2 slots x chunk x 8 bytes.  The arithmetic is
the same libnnt update kernel on the same values, so results are bitwise those of the
device-resident path.  Host logic only: every byte moves by cudaMemcpyAsync (copy engines),
every update runs in libnnt.
"""
import torch


class HostOptimizerState:
    """m (and v) for `numel` parameters in pinned host memory; `apply` streams ranges of them
    through device staging slots around an update callable."""

    def __init__(self, numel, device, two_moments=True, chunk=1 << 22):
        self.numel, self.dev = numel, torch.device(device)
        self.chunk = max(64, int(chunk) // 64 * 64)  # chunks keep the ranges' 256-byte alignment
        self.m = torch.zeros(numel, dtype=torch.float32).pin_memory()
        self.v = torch.zeros(numel, dtype=torch.float32).pin_memory() if two_moments else None
        k = 2 if two_moments else 1
        n = min(self.chunk, max(numel, 1))
        self.slots = [torch.empty(k, n, device=self.dev, dtype=torch.float32) for _ in range(2)]
        self.h2d = torch.cuda.Stream(device=self.dev)
        self.d2h = torch.cuda.Stream(device=self.dev)
        self.ev_in = [torch.cuda.Event() for _ in range(2)]
        self.ev_done = [torch.cuda.Event() for _ in range(2)]
        self.ev_free = [torch.cuda.Event() for _ in range(2)]
        self.bytes_moved = 0  # host<->device bytes of the last apply()

    def chunks(self, ranges):
        for (a, b) in ranges:
            for c in range(a, b, self.chunk):
                yield c, min(b, c + self.chunk)

    def apply(self, ranges, update, stream=None):
        """For every chunk [a, b) of the state ranges: copy m[a:b] (and v) in, call
        update(a, b, m_dev, v_dev) on `stream` (device views of the chunk's state, updated in
        place), copy them back.  Enqueued work only; `stream` waits for the last write-back."""
        stream = stream or torch.cuda.current_stream(self.dev)
        self.h2d.wait_stream(stream)  # joins the copy streams to the caller's work (and to a capture)
        self.d2h.wait_stream(stream)
        moved = 0
        for i, (a, b) in enumerate(self.chunks(ranges)):
            s, n = i % 2, b - a
            slot = self.slots[s]
            if i >= 2:
                self.h2d.wait_event(self.ev_free[s])  # the slot's previous chunk is written back
            with torch.cuda.stream(self.h2d):
                slot[0, :n].copy_(self.m[a:b], non_blocking=True)
                if self.v is not None:
                    slot[1, :n].copy_(self.v[a:b], non_blocking=True)
                self.ev_in[s].record(self.h2d)
            stream.wait_event(self.ev_in[s])
            with torch.cuda.stream(stream):
                update(a, b, slot[0, :n], slot[1, :n] if self.v is not None else None)
                self.ev_done[s].record(stream)
            self.d2h.wait_event(self.ev_done[s])
            with torch.cuda.stream(self.d2h):
                self.m[a:b].copy_(slot[0, :n], non_blocking=True)
                if self.v is not None:
                    self.v[a:b].copy_(slot[1, :n], non_blocking=True)
                self.ev_free[s].record(self.d2h)
            moved += 2 * n * 4 * (2 if self.v is not None else 1)
        stream.wait_stream(self.d2h)
        stream.wait_stream(self.h2d)
        self.bytes_moved = moved


class HostActivations:
    """The saved-activation workspaces of the first `n_layers` blocks in pinned host memory
    (tiles that do not fit the GPU live in host RAM).

    Such a layer's forward writes its `saved` workspace (LayerNorm statistics, h1, qkv, P, O, x1,
    h2, u, g: the tensors its backward reads) into one of two device slots; the copy engine then
    moves it to host RAM (device-to-host stream) while the next layers compute.  The backward
    brings it back (host-to-device stream) into the same slot, issued as soon as the slot's
    previous user (the layer two above) is done, so the transfer overlaps the backward of the
    layer in between.  The two highest offloaded layers skip the round trip: their slots still
    hold their data when the backward reaches them.  Every byte moves by cudaMemcpyAsync; the blocks'
    arithmetic is unchanged, so results are bitwise those of the resident path."""

    def __init__(self, n_layers, saved_bytes, device):
        self.n, self.dev = n_layers, torch.device(device)
        self.host = [torch.empty(saved_bytes, dtype=torch.uint8).pin_memory() for _ in range(n_layers)]
        self.slots = [torch.empty(saved_bytes, device=self.dev, dtype=torch.uint8) for _ in range(min(2, n_layers))]
        self.h2d = torch.cuda.Stream(device=self.dev)
        self.d2h = torch.cuda.Stream(device=self.dev)
        self.ev_fwd = [torch.cuda.Event() for _ in range(n_layers)]      # layer's forward done
        self.ev_bwd = [torch.cuda.Event() for _ in range(n_layers)]      # layer's backward done
        self.ev_out = [torch.cuda.Event() for _ in range(2)]             # slot's D2H copy done
        self.ev_in = [torch.cuda.Event() for _ in range(n_layers)]       # layer's H2D copy done
        self.bytes_per_layer = saved_bytes

    def slot(self, l):
        return self.slots[l % 2]

    # ---------------------------------------------------------------- forward
    def begin(self, stream):
        """Join the copy streams to the caller's work (and to a CUDA-graph capture in progress)."""
        self.h2d.wait_stream(stream)
        self.d2h.wait_stream(stream)

    def before_fwd(self, l, stream):
        """The compute stream may overwrite slot l % 2 once its previous layer's copy-out is done."""
        if l >= 2:
            stream.wait_event(self.ev_out[l % 2])

    def after_fwd(self, l, stream):
        """Copy layer l's saved workspace to host RAM (overlaps the next layers' forward)."""
        self.ev_fwd[l].record(stream)
        self.d2h.wait_event(self.ev_fwd[l])
        with torch.cuda.stream(self.d2h):
            self.host[l].copy_(self.slot(l), non_blocking=True)
            self.ev_out[l % 2].record(self.d2h)

    # ---------------------------------------------------------------- backward
    def prefetch(self, l, after_bwd_of=None):
        """Bring layer l's saved workspace back into slot l % 2 once the slot's current user (the
        backward of layer `after_bwd_of`, or the copy-out of the forward) is done."""
        if l < 0 or l >= self.n - 2:
            return  # the top two offloaded layers' slots still hold their data
        if after_bwd_of is not None:
            self.h2d.wait_event(self.ev_bwd[after_bwd_of])
        self.h2d.wait_event(self.ev_out[l % 2])
        with torch.cuda.stream(self.h2d):
            self.slot(l).copy_(self.host[l], non_blocking=True)
            self.ev_in[l].record(self.h2d)

    def before_bwd(self, l, stream):
        if l < self.n - 2:
            stream.wait_event(self.ev_in[l])

    def after_bwd(self, l, stream):
        self.ev_bwd[l].record(stream)

    def join(self, stream):
        stream.wait_stream(self.h2d)
        stream.wait_stream(self.d2h)

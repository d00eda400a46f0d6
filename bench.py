#!/usr/bin/env python
"""Benchmark: GPT-2 training step (fwd + bwd + Adam) on 1..8 B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config small] [--model gpt2|blocks]
                    [--impl nnt|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1: NCCL, one rank per GPU)

Metric (BASELINE.json): GPT-2 train tokens/s (+ model TFLOP/s, % of bf16 peak).
A step = one pass of the whole hot path over one synthetic batch per GPU.  --model gpt2
(default for small / large / xl): token + position embedding, L pre-LN GPT-2 blocks, final
LayerNorm, tied LM head over the 50257-token vocabulary, mean cross-entropy, the backward of
all of it, the DP gradient all-reduce (N > 1) and Adam on every parameter.  --model blocks
(default for wide / tiny): the L blocks with a linear-probe loss.  Weak scaling: each GPU
holds B = 8 sequences of S = 1024 tokens.  The per-step working set (activations of every
layer, GBs) is far larger than the 126 MB L2, so no explicit flush is needed between steps.

--impl reference times the CPU oracle (oracle/, fp64 NumPy) on the box's host cores on a
bounded sample of the same workload (one block over one sequence, plus the shell for gpt2).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

CONFIGS = {  # name -> (L, E, H, S, B per GPU)
    "tiny": (1, 64, 2, 32, 2),
    "small": (12, 768, 12, 1024, 8),
    "large": (36, 1280, 20, 1024, 8),
    "xl": (48, 1600, 25, 1024, 8),
    "wide": (1, 8192, 128, 1024, 8),
}
METRIC = "GPT-2 train tokens/s & model TFLOP/s at 1/2/4/8 B200; % of bf16 peak"
VOCAB = 50257  # GPT-2 BPE vocabulary (the full model: --model gpt2)


def default_model(config):
    """Full GPT-2 (embeddings + blocks + final LN + tied LM head + cross-entropy) for the named GPT-2
    sizes; the block stack for the single-layer 'wide' shape and the fp32 parity config."""
    return "blocks" if config in ("wide", "tiny") else "gpt2"


def model_flops_per_step(L, E, S, T, V=0):
    """6 N T + 12 L S E T with N = 12 E^2 per layer (full attention counted), plus 6 E V T for the
    (tied) LM head when the full model runs (PaLM / nanoGPT convention)."""
    return L * T * (72 * E * E + 12 * S * E) + 6 * E * V * T


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return dict(hbm=d["hbm_gbs"], bf16=d["bf16_tflops"], bf16_sus=d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                    src="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="fallback")


def load_traffic(config, kclass):
    """DRAM bytes per launch of kclass from the newest committed one-step ncu capture
    (profiles/r<NN>_traffic_<config>.json, written by tools/traffic.py)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_traffic_{config}.json")))
    if not files:
        return None, None
    with open(files[-1]) as f:
        d = json.load(f)
    c = d["classes"].get(kclass)
    if c is None:
        return None, None
    return c["dram_bytes_per_launch"], os.path.relpath(files[-1], ROOT) + ": " + d["source"]


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except (FileNotFoundError, OSError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        sm, mx, reasons, power = [], [], set(), []
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        with open(self.f.name) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx.append(float(parts[2]))
                    power.append(float(parts[3]))
                except ValueError:
                    continue
                for n, v in zip(names, parts[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
        os.unlink(self.f.name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "power_w_max": max(power),
                "samples": len(sm), "reasons": sorted(reasons)}


# ---------------------------------------------------------------- CPU oracle timing
def oracle_block_sample(E, H, S, seq=1, reps=None, budget_s=15.0):
    """Time the oracle (as it stands) on one block fwd+bwd+Adam over `seq` sequences of S tokens."""
    import nnt_inputs
    from oracle import dense
    P = {k: v.astype(np.float64) for k, v in nnt_inputs.make_params(E, seed=1234, init="gpt2").items()}
    x = nnt_inputs.make_x(E, S, 0, seq, seed=1001).astype(np.float64)
    r = nnt_inputs.make_r(E, S, 0, seq, seed=1001).astype(np.float64)

    def one():
        y, cache = dense.block_fwd(P, x, H)
        dense.probe_loss(y, r, seq * S)
        _, g = dense.block_bwd(P, cache, dense.probe_loss_grad(r, seq * S))
        for k in P:
            dense.adam_step(P[k], g[k], np.zeros_like(P[k]), np.zeros_like(P[k]), 1)

    t0 = time.perf_counter()
    one()
    t1 = time.perf_counter() - t0
    n = reps if reps is not None else max(1, min(20, int(budget_s / max(t1, 1e-3))))
    times = [t1]
    for _ in range(n - 1):
        t0 = time.perf_counter()
        one()
        times.append(time.perf_counter() - t0)
    return float(np.median(times)), len(times)


def oracle_shell_sample(E, V, S, reps=1):
    """Time the oracle's GPT-2 shell alone (embedding, final LN, tied LM head, cross-entropy fwd+bwd and
    Adam on the shell parameters) over one sequence of S tokens."""
    import nnt_inputs
    from oracle import dense
    sh = nnt_inputs.make_shell_params(V, S, E, seed=1234, init="gpt2")
    model = {k: v.astype(np.float64) for k, v in sh.items()}
    model["blocks"] = []
    tok = nnt_inputs.make_ids(V, S, 0, 1, seed=1001)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        _, cache = dense.gpt2_fwd(model, tok[:, :S], tok[:, 1:], 1)
        g = dense.gpt2_bwd(model, cache)
        for k in ("wte", "wpe", "lnf_g", "lnf_b"):
            dense.adam_step(model[k], g[k], np.zeros_like(model[k]), np.zeros_like(model[k]), 1)
        times.append(time.perf_counter() - t0)
    return float(np.median(times))


def host_cores():
    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:
        n = os.cpu_count()
    threads = None
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        threads = max((i.get("num_threads", 0) for i in info), default=None)
    except Exception:
        pass
    return n, threads


def oracle_sample_shape(E):
    # bounded CPU sample: one sequence; shorter for the very wide shape
    return 1024 if E <= 1600 else 256


# ---------------------------------------------------------------- model adapters
class StackRunner:
    """The block stack with the linear-probe loss: batches are (x, r)."""

    def __init__(self, st):
        self.st, self.stack = st, st

    def step(self, batch):
        return self.st.train_step(*batch)

    def set_inputs(self, batch):
        if not hasattr(self.st, "r_buf"):
            self.st.r_buf = self.st.xs[0].new_empty(self.st.xs[0].shape)
        self.st.xs[0].copy_(batch[0])
        self.st.r_buf.copy_(batch[1])

    @property
    def model(self):
        return self.st


class GPT2Runner:
    """The full GPT-2: batches are (ids, labels) int32 [B, S]."""

    def __init__(self, gm):
        self.gm, self.stack = gm, gm.stack

    def step(self, batch):
        return self.gm.train_step(*batch)

    def set_inputs(self, batch):
        self.gm.ids.copy_(batch[0].reshape(-1))
        self.gm.labels.copy_(batch[1].reshape(-1))

    @property
    def model(self):
        return self.gm


# ---------------------------------------------------------------- arms
def run_reference(args):
    """--impl reference: the oracle as it stands, on the host cores, bounded samples of the workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    L, E, H, S, B = CONFIGS[args.config]
    mdl = args.model or default_model(args.config)
    Ss = min(S, oracle_sample_shape(E))
    for _ in range(args.warmup):
        oracle_block_sample(E, H, Ss, reps=1)
    times = []
    for _ in range(args.steps):
        t, _ = oracle_block_sample(E, H, Ss, reps=1)
        times.append(t)
    t = float(np.mean(times))
    t_shell = oracle_shell_sample(E, VOCAB, Ss) if mdl == "gpt2" else 0.0
    # one sample = one block over Ss tokens; a full-model token needs L blocks (+ the shell)
    value = Ss / (t * L + t_shell)
    cores, threads = host_cores()
    sample = (f"one block fwd+bwd+Adam, 1 sequence x {Ss} tokens, E={E}, H={H}, fp64 NumPy; tokens/s = "
              f"tokens / (L x block time" + (" + shell time (embedding, final LN, tied LM head, CE, Adam)" if
                                               mdl == "gpt2" else "") + f"), L={L}")
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * t, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"gpt2-{args.config} {mdl} fwd+bwd+Adam (oracle sample)", "layers": L,
                      "d_model": E, "heads": H, "seq_len": S},
           "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads or cores, "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return 0


def run_nnt(args):
    import torch
    import torch.distributed as dist

    import nnt_inputs
    from paper_2504_13236_b200 import model, nnt

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist.group.WORLD
    nnt.nnt_device_check(local)
    L, E, H, S, B = CONFIGS[args.config]
    if args.layers:  # capacity runs (f4): the config's layer shape, a different depth
        L = args.layers
    mdl = args.model or default_model(args.config)
    dtype = "f32" if args.config == "tiny" else "bf16"
    tile = 16 if args.config == "tiny" else 1024
    sc = model.StackConfig(L=L, E=E, H=H, S=S, B=B, tile_e=tile, tile_f=tile, tile_s=tile, tile_t=tile, dtype=dtype,
                           optimizer=args.optimizer, zero=args.zero, offload=args.offload,
                           act_offload=args.act_offload)
    layers = [nnt_inputs.make_params(E, seed=1234, layer=l, init="gpt2", n_layers=L) for l in range(L)]
    b0, b1 = nnt.nnt_partition(B * world, world, rank)  # rank r's batch tiles of the global batch
    batches = []
    if mdl == "gpt2":
        shell = nnt_inputs.make_shell_params(VOCAB, S, E, seed=1234, init="gpt2")
        gm = model.GPT2Model(sc, VOCAB, layers, shell, process_group=pg, global_tokens=B * S * world)
        runner = GPT2Runner(gm)
        for i in range(2):  # two distinct synthetic batches: ids ~ U[0, V), labels = next token
            tok = nnt_inputs.make_ids(VOCAB, S, b0, b1, seed=1000 + i)
            batches.append((torch.from_numpy(np.ascontiguousarray(tok[:, :S])).pin_memory(),
                            torch.from_numpy(np.ascontiguousarray(tok[:, 1:])).pin_memory()))
    else:
        st = model.BlockStack(sc, layers, process_group=pg, global_tokens=B * S * world)
        runner = StackRunner(st)
        for i in range(2):
            x = nnt_inputs.make_x(E, S, b0, b1, seed=1000 + i)
            r = nnt_inputs.make_r(E, S, b0, b1, seed=1000 + i)
            batches.append((torch.from_numpy(x).pin_memory(), torch.from_numpy(r).pin_memory()))
    del layers
    st = runner.stack
    mm = runner.model
    dev_batches = [(x.cuda(), r.cuda()) for x, r in batches]
    T = B * S
    peaks = load_peaks()

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    use_graph = not args.no_graph
    graph_launches = 0
    if use_graph:  # the whole step as one CUDA graph (captured launches counted once); with DP the
        # bucket all-reduces + Adam are captured on the comm stream (model.BlockStack.enable_graph)
        n_cap = nnt.nnt_launch_count()
        try:
            mm.enable_graph()
        except Exception as exc:  # NCCL capture unsupported here: the DP step stays eager
            print(f"# graph capture failed ({exc!r}); eager launches", file=sys.stderr)
            mm.graph, use_graph = None, False
            torch.cuda.synchronize()
        graph_launches = nnt.nnt_launch_count() - n_cap if use_graph else 0
    for i in range(args.warmup):
        runner.step(dev_batches[i % 2])
    torch.cuda.synchronize()

    # ---------------- timed region: device-resident inputs
    sampler = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    sampler.start()
    time.sleep(0.2)
    n0 = nnt.nnt_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.steps):
        runner.step(dev_batches[i % 2])
    e1.record()
    torch.cuda.synchronize()
    launches = nnt.nnt_launch_count() - n0 + graph_launches * args.steps
    barrier()
    clocks = sampler.stop()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    # each rank's loss is its tokens' share of the global mean (scaled by 1/T_global): the global
    # mean cross-entropy is their sum over ranks
    lt = mm.loss.detach().clone()
    if world > 1:
        dist.all_reduce(lt)
    loss = float(lt.item())

    # ---------------- per-kernel timing: CUDA events around every libnnt launch scope.  With graphs,
    # a second graph of the same step is captured with timing on (the scopes become event-record
    # nodes) and replayed, so the kernels are timed as they run in the timed region; otherwise the
    # kernels run eagerly, a spin kernel queued ahead of each step so the events bracket device
    # work only, not host launch latency.
    kt = None
    timing_mode = "eager"
    if use_graph:
        try:
            nnt.nnt_timing_enable(True)
            side, st.side = st.side, None  # kernels timed one at a time (no side-stream overlap)
            try:
                tg = mm.capture_graph()
            finally:
                st.side = side
            acc = {}
            for i in range(args.steps):
                runner.set_inputs(dev_batches[i % 2])
                tg.replay()
                st.step_count += 1
                torch.cuda.synchronize()
                for k, v in nnt.nnt_timing_read().items():
                    a = acc.setdefault(k, dict(ms=0.0, launches=0, bytes=0.0, flops=0.0))
                    for f in a:
                        a[f] += v[f]
            kt = acc
            timing_mode = "graph"
            print(f"# graph-timed kernel sum {sum(v['ms'] for v in acc.values()) / args.steps:.3f} ms/step "
                  f"(timed region {ms:.3f} ms/step)", file=sys.stderr)
            del tg
        except Exception as exc:  # event nodes unsupported: fall back to the eager pass
            print(f"# graph timing failed ({exc!r}); eager timing pass", file=sys.stderr)
            kt = None
        finally:
            nnt.nnt_timing_enable(False)
    if kt is None:
        graph, mm.graph = getattr(mm, "graph", None), None
        nnt.nnt_timing_enable(True)
        for i in range(args.steps):
            torch.cuda._sleep(int(60e6))  # ~30 ms at 2 GHz, longer than one eager step's host enqueue
            runner.step(dev_batches[i % 2])
        torch.cuda.synchronize()
        kt = nnt.nnt_timing_read()
        nnt.nnt_timing_enable(False)
        mm.graph = graph
        if graph is not None:
            st.t_dev.fill_(st.step_count)  # keep the device step counter in line with the eager steps

    # ---------------- end to end: pinned host inputs copied every step, loss read back every step
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    reader = model.LossReader(2)  # each step's loss read back one step later (pipelined D2H)
    for i in range(args.steps):
        reader.push(runner.step(batches[i % 2]))
        if i:
            lv = reader.pop()
    lv = reader.pop()
    f1.record()
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(max(f0.elapsed_time(f1), 1000 * (time.perf_counter() - t0)) / args.steps)
    h2d = sum(t.numel() * t.element_size() for t in batches[0])
    d2h = 4

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    tokens = T * world
    value = tokens / (ms / 1e3)
    mflops = model_flops_per_step(L, E, S, T, VOCAB if mdl == "gpt2" else 0) * world
    model_tflops = mflops / (ms / 1e3) / 1e12
    # roofline of the dominant kernel class
    steps = args.steps
    kernels = {}
    total_k = sum(v["ms"] for v in kt.values())
    # which measured bf16 peak: the sustained one (a multi-second soak, power-capped clocks) when the
    # step runs in that regime -- a >= 1 s timed window with the SM clock held below 90 % of its
    # maximum -- else the burst one (a kernel timed alone at full clock)
    sm, sm_max = clocks.get("sm_mhz"), clocks.get("sm_max_mhz")
    sustained = bool(sm and sm_max and ms * steps >= 1000.0 and sm < 0.9 * sm_max)
    tpeak = peaks["bf16_sus"] if sustained else peaks["bf16"]
    for k, v in kt.items():
        if v["launches"] == 0:
            continue
        tensor = k == "gemm_tc"
        ach = (v["flops"] / (v["ms"] / 1e3) / 1e12) if tensor else (v["bytes"] / (v["ms"] / 1e3) / 1e9)
        peak = tpeak if tensor else peaks["hbm"]
        kernels[k] = {"ms_per_step": v["ms"] / steps, "share": v["ms"] / total_k, "launches_per_step": v["launches"] / steps,
                      "bound": "tensor" if tensor else "hbm", "achieved": ach,
                      "unit": "TFLOP/s" if tensor else "GB/s", "frac": ach / peak}
    dom = max(kernels, key=lambda k: kernels[k]["ms_per_step"])
    d = kernels[dom]
    roof = {"kernel": dom, "bound": d["bound"], "achieved": d["achieved"],
            "peak": tpeak if d["bound"] == "tensor" else peaks["hbm"], "unit": d["unit"],
            "frac": d["frac"], "traffic": None, "traffic_source": None, "peak_source": peaks["src"] +
            ((" bf16_tflops_sustained (timed window %.2f s, SM clock median %s of %s MHz: the power-capped "
              "regime the sustained figure was measured in)" % (ms * steps / 1e3, sm, sm_max)) if sustained else
             " bf16_tflops (burst)") if d["bound"] == "tensor" else " hbm_gbs",
            "frac_vs_burst": (d["achieved"] / peaks["bf16"]) if d["bound"] == "tensor" else None,
            "frac_vs_sustained": (d["achieved"] / peaks["bf16_sus"]) if d["bound"] == "tensor" else None,
            "timing": f"CUDA events around every launch scope on its stream ({timing_mode}: "
                      + ("event nodes in a replayed copy of the step graph" if timing_mode == "graph" else
                         "eager launches behind a spin kernel") + "), K steps after the timed region",
            "share_of_step": d["share"]}
    roof["traffic"], roof["traffic_source"] = load_traffic(args.config, dom)
    out = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": dtype,
           "data": ("synthetic (seeded token ids ~ U[0, 50257), next-token labels; GPT-2 init weights)"
                    if mdl == "gpt2" else "synthetic (seeded N(0,1) activations, GPT-2 init weights)"),
           "config": {"workload": (f"gpt2-{args.config}: token+position embedding, {L} pre-LN GPT-2 blocks, final "
                                   f"LayerNorm, tied LM head (V={VOCAB}), mean cross-entropy; fwd+bwd+Adam"
                                   if mdl == "gpt2" else
                                   f"gpt2-{args.config}: {L} pre-LN GPT-2 blocks fwd+bwd+Adam (block stack, "
                                   f"linear-probe loss)"),
                      "model": f"gpt2-{args.config}" + (f"-L{L}" if args.layers else "") +
                               ("" if mdl == "gpt2" else "-blocks"), "layers": L,
                      "d_model": E, "heads": H, "vocab": VOCAB if mdl == "gpt2" else None,
                      "global_batch": B * world, "seq_len": S, "tile": tile, "parallelism": f"dp{world}" + ("-zero1" if args.zero and world > 1 else ""),
                      "optimizer": args.optimizer + (" (state offloaded to pinned host memory)" if args.offload
                                                     else ""),
                      "activation_offload_layers": args.act_offload,
                      "launch": "one CUDA graph per step" if use_graph else "eager launches",
                      "l2": "per-step working set (GBs of activations) >> 126 MB L2; no explicit flush"},
           "model_tflops": model_tflops, "model_tflops_frac_of_bf16": model_tflops / peaks["bf16"],
           "loss": loss, "gpu_launches": int(launches),
           "comm": ({"backend": dist.get_backend(pg), "world_size": dist.get_world_size(pg),
                     "collective": "bucketed SUM all-reduce of the fp32 gradients on a comm stream" +
                                   (" (ZeRO-1: reduce-scatter, all-gather of bf16 weight shadows + fp32 small "
                                    "parameters)" if args.zero else "")}
                    if world > 1 else None),
           "clocks": clocks, "roofline": roof, "kernels": kernels,
           "e2e": {"value": tokens / (e2e_ms / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                   "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms}}
    if world == 1 and not args.no_cpu_baseline:
        Ss = min(S, oracle_sample_shape(E))
        t, n = oracle_block_sample(E, H, Ss, budget_s=10.0)
        t_shell = oracle_shell_sample(E, VOCAB, Ss) if mdl == "gpt2" else 0.0
        cores, threads = host_cores()
        out["cpu_baseline"] = {"value": Ss / (t * L + t_shell), "unit": "tokens/s", "cores": threads or cores,
                               "kind": "oracle",
                               "sample": f"{n} x one block fwd+bwd+Adam over 1 sequence x {Ss} tokens (E={E}, H={H}, "
                                         f"fp64 NumPy), median {t:.2f} s" +
                                         (f", plus the shell (embedding, final LN, tied LM head, CE, Adam) once, "
                                          f"{t_shell:.2f} s" if mdl == "gpt2" else "") +
                                         f"; tokens/s = tokens / (L x block + shell), L={L}"}
    print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    # default: GPT-2 XL, the configuration BASELINE.json sweeps over 1/2/4/8 B200 and the largest
    # single-GPU one (configs[3]); small / large / wide / tiny stay selectable
    ap.add_argument("--config", default="xl", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="nnt", choices=["nnt", "reference"])
    ap.add_argument("--model", default=None, choices=["gpt2", "blocks"],
                    help="gpt2 = full model with embeddings / tied LM head / cross-entropy (default for small, "
                         "large, xl); blocks = the block stack with a linear-probe loss (default for wide, tiny)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--optimizer", default="adam", choices=["adam", "sgd"], help="adam (P:194) or sgd (momentum)")
    ap.add_argument("--zero", action="store_true", help="N>1: ZeRO-1 optimizer-state sharding (reduce-scatter, "
                    "owned-slice update, all-gather of the bf16 weight shadows + fp32 small parameters) instead of "
                    "all-reduce + replicated update")
    ap.add_argument("--offload", action="store_true", help="optimizer state in pinned host memory, streamed "
                    "through device staging slots around each update (SURVEY f4)")
    ap.add_argument("--act-offload", type=int, default=0, help="saved activations of the lowest K layers in "
                    "pinned host memory, copied out after their forward and back before their backward (SURVEY f4)")
    ap.add_argument("--layers", type=int, default=0, help="override the config's layer count (capacity runs with "
                    "--act-offload / --offload; not a BASELINE configuration)")
    ap.add_argument("--no-graph", action="store_true", help="launch every kernel eagerly (no CUDA graph)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_nnt(args)


if __name__ == "__main__":
    sys.exit(main())

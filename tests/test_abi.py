"""CPU tests of the C-ABI library (no GPU): libnnt.so loads, exports every symbol
include/nnt.h declares, the integer tile bookkeeping matches the oracle's
(oracle/tiled.py) bit for bit, argument validation fails before any CUDA call,
and the lowered tile-task DAG has the structure the STF rules imply."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import nnt_inputs
from oracle import tiled

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def nnt():
    from paper_2504_13236_b200 import build
    build.build()
    from paper_2504_13236_b200 import nnt as m
    return m


def _header_functions():
    with open(os.path.join(ROOT, "include", "nnt.h")) as f:
        src = f.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:nnt_status|int|const char\s*\*|size_t|int64_t)\s+(nnt_\w+)\s*\(", src,
                                 flags=re.M)))


def test_exports_every_declared_symbol(nnt):
    names = _header_functions()
    assert len(names) >= 25
    for n in names:
        assert hasattr(nnt.lib, n), n
    assert set(names) == set(nnt.EXPORTS)
    assert nnt.nnt_abi_version() == 1


def test_tile_grid_and_extent_bit_exact(nnt):
    rng = np.random.default_rng(0)
    for _ in range(300):
        nd = int(rng.integers(1, 5))
        shape = [int(v) for v in rng.integers(1, 5000, nd)]
        tile = [int(v) for v in rng.integers(1, 6000, nd)]
        assert nnt.nnt_tile_grid(shape, tile) == tiled.tile_grid(shape, tile)
        d, t = shape[0], tile[0]
        n = tiled.tile_grid([d], [t])[0]
        for i in {0, n - 1, n // 2}:
            assert nnt.nnt_tile_extent(d, t, i) == (tiled.tile_offset(d, t, i), tiled.tile_extent(d, t, i))
    assert nnt.nnt_tile_grid([5, 3], [2, 3]) == [3, 1]


def test_partition_bit_exact(nnt):
    for n in (0, 1, 7, 8, 64, 1001):
        for R in range(1, 9):
            for r in range(R):
                assert nnt.nnt_partition(n, R, r) == tiled.partition(n, R, r)


def test_bookkeeping_errors(nnt):
    with pytest.raises(nnt.NNTError) as e:
        nnt.nnt_tile_grid([4, 0], [2, 2])
    assert e.value.status == nnt.NNT_ERR_SHAPE
    with pytest.raises(nnt.NNTError) as e:
        nnt.nnt_tile_grid([4, 4], [2, 0])
    assert e.value.status == nnt.NNT_ERR_TILE
    with pytest.raises(nnt.NNTError) as e:
        nnt.nnt_partition(8, 2, 2)
    assert e.value.status == nnt.NNT_ERR_ARG
    with pytest.raises(nnt.NNTError):
        nnt.nnt_tile_extent(10, 4, 3)


FAKE = 1 << 20  # never dereferenced: validation must fail first


def test_gemm_validation_without_gpu(nnt):
    L = nnt.lib
    S = 0  # stream (never used)
    assert L.nnt_tile_gemm(0, 1, 64, 64, 64, None, 1.0, None, 1, 64, None, FAKE, 1, 64, None, 0.0, FAKE, 0, 64,
                           None, None, None, S) == nnt.NNT_ERR_NULL
    assert L.nnt_tile_gemm(0, 1, 0, 64, 64, None, 1.0, FAKE, 1, 64, None, FAKE, 1, 64, None, 0.0, FAKE, 0, 64,
                           None, None, None, S) == nnt.NNT_ERR_SHAPE
    assert L.nnt_tile_gemm(0, 1, 64, 64, 64, None, 1.0, FAKE, 1, 64, None, FAKE, 0, 64, None, 0.0, FAKE, 0, 64,
                           None, None, None, S) == nnt.NNT_ERR_DTYPE
    tile = (C.c_int64 * 3)(16, 0, 16)
    assert L.nnt_tile_gemm(0, 1, 64, 64, 64, None, 1.0, FAKE, 1, 64, None, FAKE, 1, 64, None, 0.0, FAKE, 0, 64,
                           None, tile, None, S) == nnt.NNT_ERR_TILE
    assert L.nnt_tile_gemm(0, 1, 64, 64, 60, None, 1.0, FAKE, 1, 60, None, FAKE, 1, 60, None, 0.0, FAKE, 0, 64,
                           None, None, None, S) == nnt.NNT_ERR_ALIGN
    assert L.nnt_tile_gemm(0, 1, 64, 64, 64, None, 1.0, FAKE, 1, 32, None, FAKE, 1, 64, None, 0.0, FAKE, 0, 64,
                           None, None, None, S) == nnt.NNT_ERR_SHAPE  # lda < K
    assert L.nnt_tile_gemm(2, 1, 64, 64, 64, None, 1.0, FAKE, 1, 64, None, FAKE, 1, 64, None, 0.0, FAKE, 0, 64,
                           None, None, None, S) == nnt.NNT_ERR_ARG
    assert "trans_a" in nnt.nnt_last_error()


def test_kernel_validation_without_gpu(nnt):
    L = nnt.lib
    assert L.nnt_maxsumexp(None, 4, 8, 8, 8, 0, 4, FAKE, 0, None) == nnt.NNT_ERR_NULL
    assert L.nnt_maxsumexp(FAKE, 4, 6, 6, 6, 0, 4, FAKE, 0, None) == nnt.NNT_ERR_ALIGN
    assert L.nnt_maxsumexp(FAKE, 4, 8, 8, 0, 0, 4, FAKE, 0, None) == nnt.NNT_ERR_TILE
    assert L.nnt_softmax(FAKE, 4, 4096, 4096, 4096, 0, 4, FAKE, FAKE, 0, 4096, None) == nnt.NNT_ERR_UNSUPPORTED
    assert L.nnt_layernorm_fwd(FAKE, 4, 0, 8, 8, FAKE, FAKE, 1e-5, FAKE, 0, 8, FAKE, FAKE, None) == nnt.NNT_ERR_SHAPE
    assert L.nnt_layernorm_fwd(FAKE, 4, 8, 8, 0, FAKE, FAKE, 1e-5, FAKE, 0, 8, FAKE, FAKE, None) == nnt.NNT_ERR_TILE
    assert L.nnt_layernorm_fwd(FAKE, 4, 8, 8, 8, FAKE, FAKE, 1e-5, FAKE, 7, 8, FAKE, FAKE, None) == nnt.NNT_ERR_DTYPE
    assert L.nnt_layernorm_bwd(FAKE, 8, FAKE, 8, FAKE, FAKE, FAKE, 4, 8, None, FAKE, 8, None, FAKE, FAKE, None, 0,
                               FAKE, 1, None) == nnt.NNT_ERR_WORKSPACE
    hp = nnt.nnt_adam_hparams(1e-3, 0.9, 0.999, 1e-8, 0.0, 0.0, 0.001, 1.0)
    assert L.nnt_adam_step(16, FAKE, FAKE, FAKE, FAKE, None, C.byref(hp), None) == nnt.NNT_ERR_ARG
    assert L.nnt_gelu_fwd(FAKE, FAKE, 3, 16, None) == nnt.NNT_ERR_DTYPE
    assert L.nnt_bias_grad(FAKE, 1, 8, 8, 8, FAKE, 0, FAKE, FAKE, 1 << 20, None) == nnt.NNT_ERR_DTYPE


def _cfg(nnt, name, dtype=None, tile=None):
    c = nnt_inputs.CONFIGS[name]
    t = tile or c.tile
    dt = dtype or c.dtype
    return c, nnt.nnt_block_cfg(c.E, c.H, c.S, c.B, t, t, t, t, 1 if dt == "bf16" else 0, 1e-5, 1)


@pytest.mark.parametrize("name", ["small", "xl", "tiny"])
def test_block_workspace_sizes(nnt, name):
    c, cfg = _cfg(nnt, name)
    saved, scratch = nnt.nnt_block_workspace_size(cfg)
    dt = 2 if c.dtype == "bf16" else 4
    T, E, F = c.T, c.E, 4 * c.E
    att = c.B * c.H * c.S * c.S
    need_saved = dt * (T * E * 3 + T * 3 * E + 2 * T * F + att) + 4 * (T * E + 4 * T + 2 * c.B * c.H * c.S)
    assert need_saved <= saved <= need_saved + 256 * 16
    # fp32 path: materialised scores + dA; bf16 path: dA only (score tiles stay on chip, R26)
    assert scratch >= (dt * att if c.dtype == "bf16" else 4 * att + dt * att)


def _expected_counts(c, tile):
    g = lambda d, t: tiled.tile_grid([d], [t])[0]  # noqa: E731
    T, E, F, S = c.T, c.E, 4 * c.E, c.S
    nt, ne, n3, nf, nq = g(T, tile), g(E, tile), g(3 * E, tile), g(F, tile), g(S, tile)
    pairs = c.B * c.H * nq * (nq + 1) // 2
    fwd = {"ln1": nt, "qkv": nt * n3 * ne, "scores": pairs, "maxsumexp": pairs, "softmax": pairs, "pv": pairs,
           "out": nt * ne * ne, "ln2": nt, "fc": nt * nf * ne, "proj": nt * ne * nf}
    if c.dtype == "bf16":  # R26: subroutine 1 fused into the score tasks (no scores tensor, no maxsumexp)
        del fwd["maxsumexp"]
    bwd = {"proj_db": nt * ne, "proj_dw": ne * nf * nt, "proj_dx": nt * nf * ne, "fc_db": nt * nf,
           "fc_dw": nf * ne * nt, "fc_dx": nt * ne * nf, "ln2_bwd": nt, "out_db": nt * ne, "out_dw": ne * ne * nt,
           "out_dx": nt * ne * ne, "softmax_bwd": c.B * c.H * nq, "att_dp": pairs, "att_dv": pairs, "att_dq": pairs,
           "att_dk": pairs, "qkv_db": nt * n3, "qkv_dw": n3 * ne * nt, "qkv_dx": nt * ne * n3, "ln1_bwd": nt}
    return fwd, bwd


@pytest.mark.parametrize("name,tile", [("tiny", 16), ("tiny", 24), ("small", 1024), ("xl", 1024)])
def test_dag_task_counts_and_levels(nnt, name, tile):
    c, cfg = _cfg(nnt, name, tile=tile)
    fwd_n, bwd_n = _expected_counts(c, tile)
    tasks, groups = nnt.nnt_block_dag_describe(cfg, 0)
    names = [nnt.OP_NAMES[g.op] for g in groups]
    assert names == list(fwd_n)                              # program order == level order
    assert [g.level for g in groups] == list(range(len(fwd_n)))  # a chain: LN1 -> ... -> PROJ
    assert {nnt.OP_NAMES[g.op]: g.n_tasks for g in groups} == fwd_n
    assert len(tasks) == sum(fwd_n.values())
    assert all(t.n_deps == 0 for t in tasks if t.op == 0)    # LN1 tasks are sources
    tasks, groups = nnt.nnt_block_dag_describe(cfg, 1)
    assert {nnt.OP_NAMES[g.op]: g.n_tasks for g in groups} == bwd_n
    lv = {nnt.OP_NAMES[g.op]: g.level for g in groups}
    bf = c.dtype == "bf16"
    # dy's bf16 copy is written by proj_db (bf16 path) -> proj_dw/dx one level later
    assert lv["proj_dw"] == lv["proj_dx"] == lv["proj_db"] + (1 if bf else 0)
    assert lv["fc_db"] == lv["fc_dw"] == lv["fc_dx"] == lv["proj_dx"] + 1
    assert lv["ln2_bwd"] == lv["fc_dx"] + 1
    if bf:  # D = rowdot(dO, O) first, then the dP GEMM emits dA directly
        assert lv["softmax_bwd"] == lv["att_dv"] == lv["out_dx"] + 1
        assert lv["att_dp"] == lv["softmax_bwd"] + 1
        assert lv["att_dq"] == lv["att_dk"] == lv["att_dp"] + 1
    else:
        assert lv["att_dp"] == lv["att_dv"] == lv["out_dx"] + 1
        assert lv["softmax_bwd"] == lv["att_dp"] + 1
        assert lv["att_dq"] == lv["att_dk"] == lv["softmax_bwd"] + 1
    assert lv["qkv_dx"] == lv["att_dq"] + 1
    assert lv["ln1_bwd"] == lv["qkv_dx"] + 1
    assert [g.level for g in groups] == sorted(g.level for g in groups)
    assert len(groups) == len(bwd_n)                         # one launch group per op
    for t in tasks:
        assert groups[t.group].op == t.op and t.level <= groups[t.group].level
    # the ops the backward may run on a side stream (weak r1 #11): exactly the DAG's sinks that write
    # only parameter gradients -- the dW GEMMs and the bias column sums that copy nothing for a later
    # op (on the bf16 path proj_db also writes dy's bf16 copy, read by proj_dw / proj_dx)
    side = {nnt.OP_NAMES[g.op] for g in groups if g.side_stream_ok}
    want = {"proj_dw", "fc_db", "fc_dw", "out_db", "out_dw", "qkv_db", "qkv_dw"} | ({"proj_db"} if not bf else set())
    assert side == want
    assert not any(g.side_stream_ok for g in nnt.nnt_block_dag_describe(cfg, 0)[1])  # forward: a chain


def test_dag_reduce_tasks_are_independent(nnt):
    """K-tile tasks of one GEMM Reduce into the same C tile: no edges between them (Reduce-Reduce free)."""
    c, cfg = _cfg(nnt, "tiny", tile=16)
    tasks, groups = nnt.nnt_block_dag_describe(cfg, 0)
    qkv = [t for t in tasks if nnt.OP_NAMES[t.op] == "qkv"]
    # each qkv task reads h1(i,k) (written by one LN1 task), W and b (no writer): exactly one dependency
    assert all(t.n_deps == 1 for t in qkv)
    ms = [t for t in tasks if nnt.OP_NAMES[t.op] == "maxsumexp"]
    assert all(t.n_deps == 1 for t in ms)   # the scores tile it reads

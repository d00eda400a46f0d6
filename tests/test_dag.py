"""Serializability fuzz of the STF tile-task graph builder (SPEC S:46 rules, S:88 property)
through the C-ABI (nnt_stf_build, host-only -- runs without a GPU).

Random programs of R / W / RW / Reduce accesses over a few handles are submitted; the library
returns every task's predecessors and level.  Checked against a Python reference:
  * exact: an edge only joins an earlier task to a later one that conflicts with it on a shared
    handle or is implied by the other edges (no false dependencies), every conflicting pair (i < j) -- anything but R/R and
    Reduce/Reduce -- is ordered (j reachable from i), and level[t] = 1 + max level of its
    predecessors (0 without);
  * serializability: executing the tasks in many random orders consistent with the edges gives
    every task the same inputs and every handle the same final value as executing them
    sequentially in submission order (R reads, W / RW overwrite with a non-commutative hash, Reduce
    adds -- commutative, so Reduce tasks may run in any order among themselves, as STARPU_REDUX
    allows).
"""
import random

import pytest

from paper_2504_13236_b200 import nnt

R, W, RW, RED = 0, 1, 2, 3
MOD = (1 << 61) - 1


def _conflict(a, b):
    return not ((a == R and b == R) or (a == RED and b == RED))


def _random_program(rng, n_handles, n_tasks, modes=(R, W, RW, RED)):
    prog = []
    for _ in range(n_tasks):
        k = rng.randint(1, min(3, n_handles))
        hs = rng.sample(range(n_handles), k)
        prog.append([(h, rng.choice(modes)) for h in hs])
    return prog


def _h(*xs):
    v = 1469598103934665603
    for x in xs:
        v = ((v ^ (x & 0xFFFFFFFFFFFF)) * 1099511628211) % MOD
    return v


def _run(prog, order, n_handles):
    val = [_h(1000 + i) for i in range(n_handles)]
    seen = {}
    for t in order:
        reads = tuple(val[h] for h, m in prog[t] if m in (R, RW))
        seen[t] = reads
        for h, m in prog[t]:
            if m == W:
                val[h] = _h(t, *reads)
            elif m == RW:
                val[h] = _h(t, val[h], *reads)
            elif m == RED:
                val[h] = (val[h] + _h(7 * t + 3, *reads)) % MOD
    return val, seen


def _random_topo(rng, deps):
    n = len(deps)
    succ = [[] for _ in range(n)]
    indeg = [len(d) for d in deps]
    for t, d in enumerate(deps):
        for p in d:
            succ[p].append(t)
    ready = [t for t in range(n) if indeg[t] == 0]
    order = []
    while ready:
        t = ready.pop(rng.randrange(len(ready)))
        order.append(t)
        for s in succ[t]:
            indeg[s] -= 1
            if indeg[s] == 0:
                ready.append(s)
    assert len(order) == n  # acyclic
    return order


def _check_structure(prog, levels, deps):
    n = len(prog)
    reach = [set() for _ in range(n)]  # predecessors, transitively
    for t in range(n):
        for p in deps[t]:
            assert p < t  # edges only point forward in submission order
            reach[t] |= reach[p] | {p}
        for p in deps[t]:
            # no false dependency: an edge joins tasks that conflict on a shared handle, or is implied
            # by the other edges (a new reduction group after a read-closed one also waits for the
            # closed group's members, which the reads already waited for)
            shared = {h: m for h, m in prog[p]}
            implied = any(p in reach[q] for q in deps[t] if q != p)
            assert implied or any(h in shared and _conflict(shared[h], m) for h, m in prog[t]), (p, t)
        assert levels[t] == (1 + max(levels[p] for p in deps[t]) if deps[t] else 0)
    for j in range(n):
        for i in range(j):
            mi = {h: m for h, m in prog[i]}
            if any(h in mi and _conflict(mi[h], m) for h, m in prog[j]):
                assert i in reach[j], (i, j, prog[i], prog[j])


@pytest.mark.parametrize("seed", range(40))
def test_stf_random_programs_serializable(seed):
    rng = random.Random(seed)
    n_handles = rng.choice([1, 2, 3, 5, 8])
    n_tasks = rng.choice([5, 12, 30, 60])
    modes = (R, W, RW, RED) if seed % 4 else (R, RED)  # some programs are all reads / reductions
    prog = _random_program(rng, n_handles, n_tasks, modes)
    levels, deps = nnt.nnt_stf_build(n_handles, prog)
    _check_structure(prog, levels, deps)
    want, want_seen = _run(prog, range(n_tasks), n_handles)
    for _ in range(25):
        got, got_seen = _run(prog, _random_topo(rng, deps), n_handles)
        assert got == want
        assert got_seen == want_seen


def test_stf_spec_examples():
    """fill(W A) then gemm(R A, R B, RW C) -> one edge; two Reduce on G -> none; R twice -> none;
    a read after a reduction group depends on every member of the group."""
    levels, deps = nnt.nnt_stf_build(3, [[(0, W)], [(0, R), (1, R), (2, RW)]])
    assert deps == [[], [0]] and levels == [0, 1]
    assert nnt.nnt_stf_build(1, [[(0, RED)], [(0, RED)]])[1] == [[], []]
    assert nnt.nnt_stf_build(1, [[(0, R)], [(0, R)]])[1] == [[], []]
    levels, deps = nnt.nnt_stf_build(1, [[(0, W)], [(0, RED)], [(0, RED)], [(0, R)], [(0, W)]])
    assert deps == [[], [0], [0], [0, 1, 2], [1, 2, 3]]
    assert levels == [0, 1, 1, 2, 3]


def test_stf_rejects_bad_programs():
    with pytest.raises(nnt.NNTError):
        nnt.nnt_stf_build(2, [[(0, R), (0, W)]])  # a handle twice in one task
    with pytest.raises(nnt.NNTError):
        nnt.nnt_stf_build(2, [[(2, R)]])  # unknown handle

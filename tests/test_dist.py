"""Multi-process tests of the 1-D block-cyclic driver (paper_1505_08115_b200/dist.py).

CPU, gloo backend, world sizes 2 and 3: every rank runs dist.factorize_local on its own
columns with the oracle-backed step engine (tests/dist_numpy_engine.py), and the
gathered (R, perm) must equal the single-process reference algorithm
(oracle.block_qr, blocked.py:175-219): identical composite permutation, R to
1e-12 ||A||, and the RNG counter advanced identically.
"""

import os
import socket
import sys
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

_HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(_HERE, ".."))
sys.path.insert(0, os.path.join(_HERE, "..", "oracle"))
sys.path.insert(0, _HERE)

from paper_1505_08115_b200.dist import BlockCyclic, plan_moves  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


# ---------------------------------------------------------------------------
# host logic
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n,b,world", [(300, 50, 2), (230, 40, 3), (100, 100, 2), (257, 16, 4)])
def test_block_cyclic_layout(n, b, world):
    lay = BlockCyclic(n, b, world)
    seen = np.zeros(n, dtype=int)
    for r in range(world):
        slots = lay.slots_from(r, 0)
        assert len(slots) == lay.n_local(r)
        for j, c in enumerate(slots):
            assert lay.locate(int(c)) == (r, j)
            seen[c] += 1
        for k0 in range(lay.nblk + 1):
            tail = lay.slots_from(r, k0)
            assert lay.n_local(r) - lay.local_from(r, k0) == len(tail)
            assert np.all(tail // b >= k0)
    assert np.all(seen == 1)


@pytest.mark.parametrize("seed", range(20))
def test_plan_moves_is_the_reference_permutation(seed):
    rng = np.random.default_rng(seed)
    n, s, b = 120, 30, 20
    chosen = rng.choice(np.arange(s, n), size=b, replace=False)
    cols = np.arange(n)
    new = cols.copy()
    for src, dst in plan_moves(chosen, s, b):
        new[dst] = cols[src]
    assert np.array_equal(new[s:s + b], chosen)          # panel = chosen, in order
    assert sorted(new) == list(range(n))                 # a permutation
    assert np.array_equal(new[:s], cols[:s])             # finished columns untouched
    assert len(plan_moves(chosen, s, b)) <= 2 * b


# ---------------------------------------------------------------------------
# world_size > 1 over gloo
# ---------------------------------------------------------------------------
def _worker(rank, world, port, a, b, p, seed, out_dir, sketch="fresh"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from dist_numpy_engine import NumpyStepEngine

        from paper_1505_08115_b200.dist import block_qr_distributed
        from paper_1505_08115_b200.hqrrp import BlockConfig, RngState, SketchConfig

        rng = RngState(seed)
        cfg = BlockConfig(b, SketchConfig(b, p, 0))
        try:
            r, perm = block_qr_distributed(a, cfg, rng, engine=NumpyStepEngine(), sketch=sketch)
            np.savez(os.path.join(out_dir, f"r{rank}.npz"), r=r, perm=perm, counter=rng.counter, err="")
        except ValueError as e:
            np.savez(os.path.join(out_dir, f"r{rank}.npz"), r=np.zeros(1), perm=np.zeros(1), counter=rng.counter,
                     err=str(e))
    finally:
        dist.destroy_process_group()


def _run(world, a, b, p, seed, sketch="fresh"):
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), a, b, p, seed, d, sketch), nprocs=world, join=True)
        return [dict(np.load(os.path.join(d, f"r{q}.npz"))) for q in range(world)]


@pytest.mark.parametrize("world,m,n,b,p", [(2, 300, 300, 50, 10), (3, 260, 230, 40, 8), (2, 180, 120, 16, 4)])
def test_distributed_matches_reference_algorithm(world, m, n, b, p):
    import randqr_oracle as orc

    a = np.random.default_rng(7).standard_normal((m, n))
    ref_rng = orc.RngState(3)
    f = orc.block_qr(a, orc.BlockConfig(b, orc.SketchConfig(b, p, 0)), ref_rng)
    outs = _run(world, a, b, p, 3)
    nrm = np.linalg.norm(a)
    for o in outs:
        assert str(o["err"]) == ""
        assert np.array_equal(o["perm"], f.perm())
        assert np.abs(o["r"] - np.triu(f.r)).max() <= 1e-12 * nrm
        assert int(o["counter"]) == ref_rng.counter
    # every rank holds the same gathered result
    for o in outs[1:]:
        assert np.array_equal(o["r"], outs[0]["r"])


@pytest.mark.parametrize("world,m,n,b,p", [(2, 300, 300, 50, 10), (3, 260, 230, 40, 8)])
def test_distributed_downdate_matches_hqrrp_oracle(world, m, n, b, p):
    """HQRRP's downdated sketch over the ranks (G1 broadcast with the panel
    factors, Y2_loc -= G1 R12_loc, Y columns moving with their matrix columns) against the
    oracle restatement block_qr_downdate: same pivots, R to 1e-12 ||A||, same RNG counter."""
    import randqr_oracle as orc

    a = np.random.default_rng(11).standard_normal((m, n))
    ref_rng = orc.RngState(3)
    f = orc.block_qr_downdate(a, orc.BlockConfig(b, orc.SketchConfig(b, p, 0)), ref_rng)
    outs = _run(world, a, b, p, 3, "downdate")
    nrm = np.linalg.norm(a)
    for o in outs:
        assert str(o["err"]) == ""
        assert np.array_equal(o["perm"], f.perm())
        assert np.abs(o["r"] - np.triu(f.r)).max() <= 1e-12 * nrm
        assert int(o["counter"]) == ref_rng.counter == m * (b + p)


def test_distributed_value_error_like_reference():
    import randqr_oracle as orc

    m, n, b, p = 120, 100, 40, 30  # second panel pivots 60 columns with a 70-wide sketch
    a = np.random.default_rng(1).standard_normal((m, n))
    ref_rng = orc.RngState(5)
    with pytest.raises(ValueError):
        orc.block_qr(a, orc.BlockConfig(b, orc.SketchConfig(b, p, 0)), ref_rng)
    outs = _run(2, a, b, p, 5)
    for o in outs:
        assert "exceeds" in str(o["err"])
        assert int(o["counter"]) == ref_rng.counter

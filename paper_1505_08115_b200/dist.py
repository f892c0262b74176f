"""Multi-GPU HQRRP: 1-D block-cyclic column panels over torch.distributed ranks.

SURVEY section 8(e).  Physical column *slots* are grouped in blocks of b; slot
block k lives on rank k % G (as its local block k // G, stored contiguously in
column-major order).  Per panel i (columns s = i*b ..), with owner o = i % G:

1. every rank sketches its own trailing columns, Y_loc = Omega^T A_loc[s:, trailing]
   (blocked.py:164-172, pivoting.py:80-111; every rank draws the same Omega from
   the same counter-based stream, so Omega is never sent);
2. one all-gather of Y; every rank runs the identical column-pivoted QR of Y
   (pivoting.py:114-129), so the pivot list agrees everywhere with no second
   exchange;
3. the <= 2b moved columns travel at full height between ranks (packed per rank
   pair, batched send/recv); the rest of the matrix never moves;
4. the owner factors the panel (qr_tall_pivoted, householder.py:183-198) and
   broadcasts V, T, Q2 and P-hat in one message;
5. every rank applies the panel to its own trailing columns
   (householder.py:105-114).

Host bookkeeping -- which original column sits in each slot, and its logical
position, which decides the reference's ties and "rest in original order"
(pivoting.py:125-128) -- is replicated and updated identically on every rank.
After the last panel the slots hold R's columns in the reference's order, so
``perm[slot]`` is the reference's composite permutation.

Device work goes through an *engine*; the product engine is ``CudaStepEngine``
(the C ABI's panel-step entry points).  Collectives are torch.distributed calls
(NCCL between GPUs).  Fresh or downdated sketches (``sketch=``), q = 0, permutation
pivots and m >= n are supported; power iterations, reflector pivots and block_rrqr run on
one GPU (hqrrp.block_qr / block_rrqr).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from .errors import DimensionError, check
from .hqrrp import BlockConfig, Engine, RngState


def _ptr(t, off=0, esize=8):
    return ctypes.c_void_p(t.data_ptr() + esize * off)


class _Ready:
    """Selection result already on the host (CPU engines)."""

    def __init__(self, v):
        self.v = v

    def result(self):
        return self.v


class _PendingSelect:
    """Pivots copied to pinned host memory behind an event: ``result()`` waits for the
    selection only, not for the trailing update enqueued after it (look-ahead)."""

    def __init__(self, host, event):
        self.host, self.event = host, event

    def result(self):
        self.event.synchronize()
        return self.host.numpy().astype(np.int64)


def _host_index(torch, arr, device):
    """int64 index tensor on `device` from host data, without synchronising the stream
    (pinned staging + non-blocking copy; CPU devices get the tensor directly)."""
    t = torch.from_numpy(np.ascontiguousarray(np.asarray(arr, dtype=np.int64)))
    if device.type != "cuda":
        return t
    return t.pin_memory().to(device, non_blocking=True)


class CudaStepEngine:
    """Panel steps on the GPU through the C ABI (rq_gemm, rq_sketch_select,
    rq_panel_factor, rq_panel_apply, rq_householder_sweep, rq_gaussian_matrix)."""

    defer_rest = os.environ.get("RQ_DIST_DEFER", "0") == "1"

    def __init__(self, engine: Engine | None = None):
        import torch

        self.torch = torch
        self.eng = engine if engine is not None else Engine()
        self.lib = self.eng.lib
        self.h = self.eng.handle
        self.device = self.eng.device

    # storage convention: column-major rows x cols, tensor of shape (cols, ld), ld even
    def alloc(self, rows, cols):
        buf, ld = self.eng.alloc_matrix(rows, cols)
        buf.zero_()
        return buf, ld

    def gaussian(self, rows, cols, seed, counter):
        buf, ld = self.alloc(rows, cols)
        check(self.lib.rq_gaussian_matrix(self.h, rows, cols, seed, counter, _ptr(buf), ld))
        return buf, ld

    def sketch(self, om, ldo, a, lda, a_rows, a_cols, r0, c0, mp, nt, wdt, cols_alloc):
        y, ldy = self.alloc(wdt, max(cols_alloc, 1))
        if nt > 0:
            check(self.lib.rq_gemm(self.h, 0, wdt, nt, mp, _ptr(om), ldo, mp, wdt, 0, 0, _ptr(a), lda, a_rows,
                                   a_cols, r0, c0, _ptr(y), ldy, 1.0, 0.0))
        return y, ldy

    def index(self, arr):
        return _host_index(self.torch, arr, self.device)

    def select_async(self, y, ldy, wdt, n, steps, init_pos):
        torch = self.torch
        ip = _host_index(torch, init_pos, self.device).to(torch.int32)
        ch = torch.empty(steps, dtype=torch.int32, device=self.device)
        check(self.lib.rq_sketch_select(self.h, _ptr(y), ldy, wdt, n, steps, _ptr(ip), _ptr(ch)))
        host = torch.empty(steps, dtype=torch.int32, pin_memory=True)
        host.copy_(ch, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(self.eng.stream)
        return _PendingSelect(host, ev)

    def select(self, y, ldy, wdt, n, steps, init_pos):
        return self.select_async(y, ldy, wdt, n, steps, init_pos).result()

    def panel_factor(self, p, ldp, mp, b):
        torch = self.torch
        v, ldv = self.alloc(mp, b)
        t, ldt = self.alloc(b, b)
        q2, ldq = self.alloc(b, b)
        ph = torch.empty(b, dtype=torch.int32, device=self.device)
        check(self.lib.rq_panel_factor(self.h, _ptr(p), ldp, mp, b, _ptr(v), ldv, _ptr(t), ldt, _ptr(q2), ldq,
                                       _ptr(ph)))
        return (v, ldv, t, ldt, q2, ldq), ph.to(torch.int64)

    def panel_apply(self, fac, mp, b, a, lda, a_rows, a_cols, r0, c0, n2):
        v, ldv, t, ldt, q2, ldq = fac
        check(self.lib.rq_panel_apply(self.h, _ptr(v), ldv, _ptr(t), ldt, _ptr(q2), ldq, mp, b, _ptr(a), lda,
                                      a_rows, a_cols, r0, c0, n2))

    def panel_apply_top(self, fac, mp, b, a, lda, a_rows, a_cols, r0, c0, n2):
        """The rows the next panel's pivots depend on (look-ahead): W = V^T A2, W2 = T^T W,
        A2[0:b] -= V[0:b] W2, then Q2^T on those rows; returns W2 for panel_apply_rest."""
        v, ldv, t, ldt, q2, ldq = fac
        w, ldw = self.alloc(b, n2)
        w2, _ = self.alloc(b, n2)
        g = self.lib.rq_gemm
        check(g(self.h, 0, b, n2, mp, _ptr(v), ldv, mp, b, 0, 0, _ptr(a), lda, a_rows, a_cols, r0, c0, _ptr(w), ldw,
                1.0, 0.0))
        check(g(self.h, 0, b, n2, b, _ptr(t), ldt, b, b, 0, 0, _ptr(w), ldw, b, n2, 0, 0, _ptr(w2), ldw, 1.0, 0.0))
        c = _ptr(a, c0 * lda + r0)
        check(g(self.h, 1, b, n2, b, _ptr(v), ldv, mp, b, 0, 0, _ptr(w2), ldw, b, n2, 0, 0, c, lda, -1.0, 1.0))
        w[:n2, :b] = a[c0:c0 + n2, r0:r0 + b]
        check(g(self.h, 0, b, n2, b, _ptr(q2), ldq, b, b, 0, 0, _ptr(w), ldw, b, n2, 0, 0, c, lda, 1.0, 0.0))
        return w2, ldw

    def panel_apply_rest(self, fac, top, mp, b, a, lda, a_rows, a_cols, r0, c0, n2, w_off=0, h=None):
        """A2[b:] -= V[b:] W2 (the trailing update below the panel's rows); W2's columns start at
        w_off (a sub-range of the local trailing columns)."""
        v, ldv, t, ldt, q2, ldq = fac
        w2, ldw = top
        if mp > b and n2 > 0:
            check(self.lib.rq_gemm(h or self.h, 1, mp - b, n2, b, _ptr(v), ldv, mp, b, b, 0, _ptr(w2), ldw, b,
                                   w2.shape[0], 0, w_off, _ptr(a, c0 * lda + r0 + b), lda, -1.0, 1.0))

    # ---- deferred rest of the update (look-ahead): the columns the next exchange / panel
    #      needs first (gathered), then the bulk on a side stream beside the next panel ----
    def panel_apply_rest_cols(self, fac, top, mp, b, a, lda, r0, t1, cols):
        if mp <= b or len(cols) == 0:
            return
        torch = self.torch
        w2, ldw = top
        idx = self.index(cols)
        widx = self.index(np.asarray(cols) - t1)
        k = len(cols)
        x, ldx = self.alloc(mp - b, k)
        x[:k, :mp - b] = a.index_select(0, idx)[:, r0 + b:r0 + mp]
        ws, ldws = self.alloc(b, k)
        ws[:k, :b] = w2.index_select(0, widx)[:, :b]
        v = fac[0]
        check(self.lib.rq_gemm(self.h, 1, mp - b, k, b, _ptr(v), fac[1], mp, b, b, 0, _ptr(ws), ldws, b, k, 0, 0,
                               _ptr(x), ldx, -1.0, 1.0))
        rows = a.index_select(0, idx)
        rows[:, r0 + b:r0 + mp] = x[:k, :mp - b]
        a.index_copy_(0, idx, rows)
        w2.index_fill_(0, widx, 0.0)

    def zero_cols(self, top, cols):
        if len(cols):
            top[0].index_fill_(0, self.index(cols), 0.0)

    def _side(self):
        if getattr(self, "_side_eng", None) is None:
            st = self.torch.cuda.Stream(device=self.device)
            self._side_eng = Engine(self.device.index, stream=st)
            # its GEMMs leave 16 SMs to the panel's cluster kernels on the main stream
            check(self.lib.rq_ctx_set_gemm_cap(self._side_eng.handle, 148 - 16))
        return self._side_eng

    def rest_async(self, fac, top, mp, b, a, lda, a_rows, a_cols, r0, c0, n2, w_off, keep):
        """panel_apply_rest on a side stream (its own library context); returns the event the
        main stream waits for before the next panel's trailing update."""
        torch = self.torch
        se = self._side()
        ev0 = torch.cuda.Event()
        ev0.record(self.eng.stream)
        se.stream.wait_event(ev0)
        with torch.cuda.stream(se.stream):
            self.panel_apply_rest(fac, top, mp, b, a, lda, a_rows, a_cols, r0, c0, n2, w_off, h=se.handle)
            for t in keep:  # main-stream tensors the side stream reads: not reused before it is done
                t.record_stream(se.stream)
            top[0].record_stream(se.stream)
        ev1 = torch.cuda.Event()
        ev1.record(se.stream)
        return ev1

    def wait(self, ev):
        if ev is not None:
            self.eng.stream.wait_event(ev)

    def downdate_g1(self, y, ldy, wdt, c0, ph, p, ldp, b, g1, ldg):
        """G1 = Y1 R11^{-1} (written into g1, wdt x b): Y1 = the panel's sketch columns c0.. of y
        in P-hat order, R11 = the factored panel's top b x b (downdated sketch)."""
        torch = self.torch
        y1, ldy1 = self.alloc(wdt, b)
        y1[:b, :wdt].copy_(y[c0:c0 + b, :wdt].index_select(0, ph.to(torch.int64)))
        x, ldx = self.alloc(b, b)
        check(self.lib.rq_trinv_upper(self.h, _ptr(p), ldp, b, _ptr(x), ldx))
        check(self.lib.rq_gemm(self.h, 1, wdt, b, b, _ptr(y1), ldy1, wdt, b, 0, 0, _ptr(x), ldx, b, b, 0, 0,
                               _ptr(g1), ldg, 1.0, 0.0))

    def downdate_apply(self, g1, ldg, wdt, b, a, lda, a_rows, a_cols, s, t1, n2, y, ldy):
        """Y2 <- Y2 - G1 R12 on the local columns t1 .. t1+n2 (R12 = their final top rows s..s+b)."""
        if n2 <= 0:
            return
        check(self.lib.rq_gemm(self.h, 1, wdt, n2, b, _ptr(g1), ldg, wdt, b, 0, 0, _ptr(a), lda, a_rows, a_cols, s,
                               t1, _ptr(y[t1:]), ldy, -1.0, 1.0))

    def final_block(self, blk, ldb, mp, w):
        """Column-pivoted sweep of an mp x w block in place; returns perm (position t holds column perm[t])."""
        torch = self.torch
        v, ldv = self.alloc(mp, w)
        perm = torch.arange(w, dtype=torch.int64, device=self.device)
        check(self.lib.rq_householder_sweep(self.h, _ptr(blk), mp, w, ldb, _ptr(v), ldv, _ptr(perm), min(mp, w), 1))
        return perm

    def synchronize(self):
        self.torch.cuda.synchronize(self.device)


# --------------------------------------------------------------------------
# 1-D block-cyclic layout of the column slots
# --------------------------------------------------------------------------
@dataclass
class BlockCyclic:
    n: int
    b: int
    world: int

    @property
    def nblk(self):
        return -(-self.n // self.b)

    def size(self, k):
        return min(self.b, self.n - k * self.b)

    def owner(self, k):
        return k % self.world

    def local_off(self, k):
        """Local column offset of slot block k on its owner (every block but the last is full)."""
        return (k // self.world) * self.b

    def n_local(self, r):
        return sum(self.size(k) for k in range(r, self.nblk, self.world))

    def first_owned(self, r, k0):
        """First block index >= k0 owned by rank r, or None."""
        k = k0 + ((r - k0) % self.world)
        return k if k < self.nblk else None

    def local_from(self, r, k0):
        """Local column offset where rank r's blocks k >= k0 start (n_local if none)."""
        k = self.first_owned(r, k0)
        return self.n_local(r) if k is None else self.local_off(k)

    def slots_from(self, r, k0):
        """Physical slots of rank r's blocks k >= k0, in local storage order."""
        k = self.first_owned(r, k0)
        if k is None:
            return np.zeros(0, dtype=np.int64)
        return np.concatenate([np.arange(kk * self.b, kk * self.b + self.size(kk), dtype=np.int64)
                               for kk in range(k, self.nblk, self.world)])

    def locate(self, slot):
        """(owner rank, local column) of a physical slot."""
        k = slot // self.b
        return self.owner(k), self.local_off(k) + (slot - k * self.b)


def plan_moves(chosen_slots, s, b):
    """Full-height column moves that put the chosen slots' columns into slots s..s+b-1
    (in selection order) and the displaced panel columns into the vacated slots.
    Returns a list of (src_slot, dst_slot)."""
    chosen = [int(c) for c in chosen_slots]
    cset = set(chosen)
    moves = [(c, s + t) for t, c in enumerate(chosen) if c != s + t]
    displaced = [d for d in range(s, s + b) if d not in cset]
    vacated = [c for c in chosen if c >= s + b]
    assert len(displaced) == len(vacated)
    moves += list(zip(displaced, vacated))
    return moves


def _apply_moves_host(arr, moves):
    old = arr.copy()
    for src, dst in moves:
        arr[dst] = old[src]


class _Dist:
    def __init__(self, group):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.world = dist.get_world_size(group)
            self.rank = dist.get_rank(group)
        else:  # single process without a process group (e.g. the fp32 path on one GPU)
            self.world = 1
            self.rank = 0

    def global_rank(self, r):
        if self.group is None:
            return r
        return self.dist.get_global_rank(self.group, r)


def _exchange_columns(a_loc, m, lay, rank, moves, d: _Dist, engine):
    """Execute full-height column moves between ranks: gather every outgoing column
    first, then write every incoming one (so a slot can be both source and target)."""
    torch = engine.torch
    world = d.world
    send = {q: [] for q in range(world)}  # (move index, local src col) per destination rank
    recv = {q: [] for q in range(world)}  # (move index, local dst col) per source rank
    for idx, (src, dst) in enumerate(moves):
        rs, ls = lay.locate(src)
        rd, ldst = lay.locate(dst)
        if rs == rank:
            send[rd].append((idx, ls))
        if rd == rank:
            recv[rs].append((idx, ldst))
    bufs_out = {}
    for q, lst in send.items():
        if lst:
            cols = _host_index(torch, [c for _, c in lst], a_loc.device)
            bufs_out[q] = a_loc.index_select(0, cols).contiguous()
    bufs_in = {}
    for q, lst in recv.items():
        if lst:
            bufs_in[q] = bufs_out[q] if q == rank else torch.empty((len(lst), a_loc.shape[1]), dtype=a_loc.dtype,
                                                                   device=a_loc.device)
    ops = []
    for q in range(world):
        if q == rank:
            continue
        if q in bufs_out:
            ops.append(d.dist.P2POp(d.dist.isend, bufs_out[q], d.global_rank(q), d.group))
        if q in bufs_in:
            ops.append(d.dist.P2POp(d.dist.irecv, bufs_in[q], d.global_rank(q), d.group))
    if ops:
        for req in d.dist.batch_isend_irecv(ops):
            req.wait()
    for q, lst in recv.items():
        if lst:
            cols = _host_index(torch, [c for _, c in lst], a_loc.device)
            a_loc.index_copy_(0, cols, bufs_in[q])


@dataclass
class DistResult:
    """Local result of one rank: R's columns in this rank's slots, plus the global perm."""

    a_loc: object      # storage (n_loc, lda): R's columns of the owned slots
    lda: int
    m: int
    n: int
    layout: BlockCyclic
    perm: np.ndarray   # perm[j] = original column at position j (A[:, perm] = Q R)


def factorize_local(a_loc, lda, m, n, cfg: BlockConfig, rng: RngState, *, group=None, engine=None,
                    sketch: str = "fresh"):
    """HQRRP (permutation pivots) on this rank's block-cyclic columns.

    ``sketch="fresh"`` draws a new Omega per panel (the reference's semantics);
    ``sketch="downdate"`` is HQRRP's downdated sketch: G is drawn once
    (counter += m (b+p)), Y_loc = G A_loc, the Y columns travel with their matrix columns, and
    after each panel every rank updates its own columns Y2_loc -= G1 R12_loc with
    G1 = Y1 R11^{-1} broadcast by the panel's owner together with V, T, Q2 and P-hat.

    ``a_loc`` is the (n_local, lda) column-major storage of the slot blocks this rank
    owns (see ``BlockCyclic``); it is overwritten with the rank's columns of R.
    ``rng.counter`` advances exactly as in the single-GPU / reference run."""
    d = _Dist(group)
    engine = engine if engine is not None else CudaStepEngine()
    torch = engine.torch
    b = cfg.block
    sk = cfg.resolved_sketch()
    if cfg.pivot_kind != "permutation" or cfg.rrqr:
        raise NotImplementedError("multi-GPU path: permutation pivots (block_qr) only")
    if sk.power != 0:
        raise NotImplementedError("multi-GPU path: power iterations run on one GPU")
    if m < n:
        raise DimensionError(f"blocked QR needs rows >= cols, got {m}x{n}")
    if b < 1 or b > n:
        raise DimensionError(f"block size must lie in [1, {n}], got {b}")
    wdt = b + sk.oversample
    lay = BlockCyclic(n, b, d.world)
    rank = d.rank
    nloc = lay.n_local(rank)
    if a_loc.shape[0] < nloc or lda < m:
        raise DimensionError("local storage does not hold this rank's columns")
    # the reference raises before drawing the offending sketch (pivoting.py:97-98)
    for s in range(0, n, b):
        if n - s <= b:
            break
        if wdt > n - s:
            bad = s
            if sketch == "downdate":  # G was drawn before the loop (oracle block_qr_downdate)
                rng.counter += m * wdt
            else:
                rng.counter += sum((m - t) * wdt for t in range(0, bad, b))
            raise ValueError(f"sketch width {wdt} exceeds the {n - s} columns being pivoted")
    if sketch not in ("fresh", "downdate"):
        raise ValueError(f"sketch must be 'fresh' or 'downdate', got {sketch!r}")
    downdate = sketch == "downdate" and n > b
    al = getattr(engine, "ld_align", 2)  # the fp32 engine's tensor-core GEMMs need ld % 4 == 0
    slot_orig = np.arange(n, dtype=np.int64)
    slot_lpos = np.arange(n, dtype=np.int64)
    counts_cache = {}
    ph_pending = []
    y_loc, ldyl = None, 0
    if downdate:
        # G drawn once (the same stream on every rank), Y_loc = G A_loc
        g_om, ldgo = engine.gaussian(m, wdt, rng.seed, rng.counter)
        rng.counter += m * wdt
        y_loc, ldyl = engine.sketch(g_om, ldgo, a_loc, lda, m, nloc, 0, 0, m, nloc, wdt, nloc)
        del g_om
        ldg = (wdt + al - 1) // al * al
    def start_select(i):
        """Steps 1-2 for panel i: the local sketch columns (fresh, or the downdated Y_loc), one
        all-gather, and the identical pivot selection on every rank -- returned as a pending
        host result (the trailing update enqueued after it keeps the GPU busy meanwhile)."""
        s = i * b
        np_, mp = n - s, m - s
        counts = counts_cache.get(i)
        if counts is None:
            counts = [lay.n_local(q) - lay.local_from(q, i) for q in range(d.world)]
            counts_cache[i] = counts
        cmax = max(counts)
        t0 = lay.local_from(rank, i)
        if downdate:
            y, ldy = engine.alloc(wdt, max(cmax, 1))
            if counts[rank] > 0:
                y[:counts[rank], :wdt].copy_(y_loc[t0:t0 + counts[rank], :wdt])
        else:
            om, ldo = engine.gaussian(mp, wdt, rng.seed, rng.counter)
            rng.counter += mp * wdt
            y, ldy = engine.sketch(om, ldo, a_loc, lda, m, nloc, s, t0, mp, counts[rank], wdt, cmax)
            del om
        if d.world > 1:
            gathered = torch.empty((d.world * cmax, ldy), dtype=y.dtype, device=y.device)
            d.dist.all_gather_into_tensor(gathered, y[:cmax].contiguous(), group=d.group)
            idx = np.concatenate([np.arange(q * cmax, q * cmax + counts[q]) for q in range(d.world)])
            y_all = gathered.index_select(0, _host_index(torch, idx, y.device)).contiguous()
            del gathered
        else:
            y_all = y[:counts[0]].contiguous()
        ycol_slot = np.concatenate([lay.slots_from(q, i) for q in range(d.world)])
        init_pos = slot_lpos[ycol_slot] - s
        if hasattr(engine, "select_async"):
            fut = engine.select_async(y_all, ldy, wdt, np_, b, init_pos)
        else:
            fut = _Ready(engine.select(y_all, ldy, wdt, np_, b, init_pos))
        return fut, ycol_slot

    # Look-ahead (downdated sketch): panel i+1's pivots depend only on the
    # top b rows of panel i's trailing update (R12), so its selection is enqueued between those
    # rows and the rest of the update; the host then waits for the pivots while the GPU runs
    # the rest of the update.
    lookahead = downdate and hasattr(engine, "panel_apply_top")
    # Deferring the bulk of the update to a side stream beside the next panel's factorization
    # (rest_async) measured slower with the CUDA engines -- rq_panel_factor's WY updates between
    # leaves need the whole GPU (n = 10k, N = 1: 230 vs 199 ms) -- so they opt in (RQ_DIST_DEFER=1)
    defer_rest = lookahead and hasattr(engine, "rest_async") and getattr(engine, "defer_rest", False)
    pending = None
    deferred = None
    rest_ev = None
    for i in range(lay.nblk):
        s = i * b
        np_ = n - s
        mp = m - s
        o = lay.owner(i)
        if np_ <= b:
            if rest_ev is not None:
                engine.wait(rest_ev)
                rest_ev = None
            _apply_pending_phat(slot_orig, ph_pending)
            _final_block(a_loc, lda, m, n, s, i, lay, rank, slot_orig, slot_lpos, d, engine)
            break
        # ---- 1-2: sketch, all-gather, selection (started by the previous panel's look-ahead) ----
        if pending is None:
            pending = start_select(i)
        fut, ycol_slot = pending
        pending = None
        chosen_y = fut.result()
        chosen = ycol_slot[chosen_y]
        # ---- 3: move the chosen columns into the panel slots ----
        moves = plan_moves(chosen, s, b)
        if deferred is not None:
            # the previous panel's update below its rows: first on the columns that move and on
            # this panel's block (owner), then the bulk beside this panel's factorization
            fac_d, top_d, mp_d, s_d, t1_d, n2_d, keep_d = deferred
            deferred = None
            sent = [lay.locate(src)[1] for src, _ in moves if lay.locate(src)[0] == rank]
            recv = [lay.locate(dst)[1] for _, dst in moves if lay.locate(dst)[0] == rank]
            own = rank == o
            pre = set(sent) | (set(range(t1_d, t1_d + b)) if own else set())
            pre = sorted(c for c in pre if t1_d <= c < t1_d + n2_d)
            engine.panel_apply_rest_cols(fac_d, top_d, mp_d, b, a_loc, lda, s_d, t1_d, pre)
            engine.zero_cols(top_d, [c - t1_d for c in recv if t1_d <= c < t1_d + n2_d])
            _exchange_columns(a_loc, m, lay, rank, moves, d, engine)
            c_lo = t1_d + (b if own else 0)
            rest_ev = engine.rest_async(fac_d, top_d, mp_d, b, a_loc, lda, m, nloc, s_d, c_lo,
                                        t1_d + n2_d - c_lo, c_lo - t1_d, keep_d)
        else:
            _exchange_columns(a_loc, m, lay, rank, moves, d, engine)
        if downdate:  # the sketch columns follow their matrix columns
            _exchange_columns(y_loc, wdt, lay, rank, moves, d, engine)
        _apply_moves_host(slot_orig, moves)
        _apply_moves_host(slot_lpos, moves)
        rest = np.arange(s + b, n, dtype=np.int64)
        order = np.argsort(slot_lpos[rest], kind="stable")
        slot_lpos[rest[order]] = s + b + np.arange(rest.size, dtype=np.int64)
        slot_lpos[s:s + b] = s + np.arange(b, dtype=np.int64)
        # ---- 4: panel on the owner; V, T, Q2, P-hat broadcast in one message ----
        ldv = (mp + al - 1) // al * al
        ldb = (b + al - 1) // al * al
        nph = (b + al - 1) // al * al  # P-hat, padded so G1 after it stays 16-byte aligned
        ng1 = b * ldg if downdate else 0
        nfac = b * ldv + 2 * b * ldb + nph
        pack = torch.empty(nfac + ng1, dtype=a_loc.dtype, device=a_loc.device)  # P-hat exact in fp32 too (b < 2^24)
        if rank == o:
            lo = lay.local_off(i)
            p, ldp = engine.alloc(mp, b)
            p[:b, :mp].copy_(a_loc[lo:lo + b, s:m])
            fac, ph = engine.panel_factor(p, ldp, mp, b)
            if downdate:  # G1 = Y1 R11^{-1} from the factored panel (R11 = p's top b x b)
                g1b = pack[nfac:].view(b, ldg)
                engine.downdate_g1(y_loc, ldyl, wdt, lo, ph, p, ldp, b, g1b, ldg)
            a_loc[lo:lo + b, s:m].copy_(p[:b, :mp])
            if s > 0:  # rows above follow P-hat
                a_loc[lo:lo + b, :s] = a_loc[lo:lo + b, :s].index_select(0, ph)
            v, _, t, _, q2, _ = fac
            pack[:b * ldv].copy_(v[:b, :ldv].reshape(-1))
            pack[b * ldv:b * ldv + b * ldb].copy_(t[:b, :ldb].reshape(-1))
            pack[b * ldv + b * ldb:b * ldv + 2 * b * ldb].copy_(q2[:b, :ldb].reshape(-1))
            pack[nfac - nph:nfac - nph + b].copy_(ph.to(pack.dtype))
        if d.world > 1:
            d.dist.broadcast(pack, src=d.global_rank(o), group=d.group)
        v = pack[:b * ldv].view(b, ldv)
        t = pack[b * ldv:b * ldv + b * ldb].view(b, ldb)
        q2 = pack[b * ldv + b * ldb:b * ldv + 2 * b * ldb].view(b, ldb)
        # P-hat reorders the panel's slots; those never compete for pivots again, so only
        # the final perm needs it: keep it on the device (no host sync here), apply at the end
        ph_pending.append((s, pack[nfac - nph:nfac - nph + b].clone()))
        if hasattr(engine, "record_panel"):  # engines that form Q themselves keep the factors
            engine.record_panel(s, mp, b, (v, ldv, t, ldb, q2, ldb))
        # ---- 5: trailing update of the local columns ----
        t1 = lay.local_from(rank, i + 1)
        n2 = nloc - t1
        fac = (v, ldv, t, ldb, q2, ldb)
        next_full = n - (s + b) > b
        if lookahead:
            engine.wait(rest_ev)  # the previous panel's bulk update (side stream)
            rest_ev = None
            top = engine.panel_apply_top(fac, mp, b, a_loc, lda, m, nloc, s, t1, n2) if n2 > 0 else None
            if next_full:
                # ---- 6: Y2_loc -= G1 R12_loc, then the next panel's selection (every rank) ----
                if n2 > 0:
                    engine.downdate_apply(pack[nfac:].view(b, ldg), ldg, wdt, b, a_loc, lda, m, nloc, s, t1, n2,
                                          y_loc, ldyl)
                pending = start_select(i + 1)
            if n2 > 0:
                if next_full and defer_rest:
                    deferred = (fac, top, mp, s, t1, n2, [pack])
                else:
                    engine.panel_apply_rest(fac, top, mp, b, a_loc, lda, m, nloc, s, t1, n2)
        elif n2 > 0:
            engine.panel_apply(fac, mp, b, a_loc, lda, m, nloc, s, t1, n2)
            # ---- 6 (downdate): Y2_loc -= G1 R12_loc on the local trailing columns ----
            if downdate and next_full:
                engine.downdate_apply(pack[nfac:].view(b, ldg), ldg, wdt, b, a_loc, lda, m, nloc, s, t1, n2,
                                      y_loc, ldyl)
        del pack
    _apply_pending_phat(slot_orig, ph_pending)
    return DistResult(a_loc, lda, m, n, lay, slot_orig)


def _apply_pending_phat(slot_orig, pending):
    """slot s + t of each finished panel holds what was in slot s + P-hat[t]."""
    if not pending:
        return
    import torch

    allph = torch.stack([p for _, p in pending]).cpu().numpy().astype(np.int64)  # one sync
    for (s, _), ph in zip(pending, allph):
        slot_orig[s:s + len(ph)] = slot_orig[s + ph]
    pending.clear()


def _final_block(a_loc, lda, m, n, s, i, lay, rank, slot_orig, slot_lpos, d: _Dist, engine):
    """Last block (n - s <= b columns, one owner): reference order, then a full-height CPQR."""
    torch = engine.torch
    w = n - s
    mp = m - s
    o = lay.owner(i)
    order = np.argsort(slot_lpos[s:n], kind="stable")
    permbuf = torch.empty(w, dtype=torch.float64, device=a_loc.device)
    if rank == o:
        lo = lay.local_off(i)
        idx = torch.as_tensor(lo + order, dtype=torch.int64, device=a_loc.device)
        a_loc[lo:lo + w] = a_loc.index_select(0, idx)
        blk, ldb = engine.alloc(mp, w)
        blk[:w, :mp].copy_(a_loc[lo:lo + w, s:m])
        perm = engine.final_block(blk, ldb, mp, w)
        a_loc[lo:lo + w, s:m].copy_(blk[:w, :mp])
        if s > 0:
            a_loc[lo:lo + w, :s] = a_loc[lo:lo + w, :s].index_select(0, perm)
        permbuf.copy_(perm.to(torch.float64))
    if d.world > 1:
        d.dist.broadcast(permbuf, src=d.global_rank(o), group=d.group)
    perm_host = permbuf.cpu().numpy().astype(np.int64)
    slot_orig[s:n] = slot_orig[s + order]
    slot_orig[s:n] = slot_orig[s + perm_host]
    slot_lpos[s:n] = np.arange(s, n)


# --------------------------------------------------------------------------
# Convenience: scatter a full matrix, factorize, gather R on every rank
# --------------------------------------------------------------------------
def scatter_columns(a_full_storage, m, n, b, world, rank, engine):
    """This rank's block-cyclic columns of a full (n, ld) column-major storage."""
    lay = BlockCyclic(n, b, world)
    slots = lay.slots_from(rank, 0)
    buf, lda = engine.alloc(m, max(len(slots), 1))
    if len(slots):
        idx = engine.torch.as_tensor(slots, dtype=engine.torch.int64, device=buf.device)
        buf[:len(slots), :m].copy_(a_full_storage.index_select(0, idx)[:, :m])
    return buf, lda


def gather_r(res: DistResult, engine, group=None):
    """R (n-column storage (n, lda), reference order) assembled on every rank."""
    d = _Dist(group)
    torch = engine.torch
    lay = res.layout
    counts = [lay.n_local(q) for q in range(d.world)]
    cmax = max(counts)
    local = torch.zeros((cmax, res.lda), dtype=res.a_loc.dtype, device=res.a_loc.device)
    local[:counts[d.rank]].copy_(res.a_loc[:counts[d.rank], :res.lda])
    if d.world > 1:
        allb = torch.empty((d.world * cmax, res.lda), dtype=local.dtype, device=local.device)
        d.dist.all_gather_into_tensor(allb, local, group=d.group)
    else:
        allb = local
    full = torch.zeros((res.n, res.lda), dtype=local.dtype, device=local.device)
    for q in range(d.world):
        slots = lay.slots_from(q, 0)
        if len(slots):
            full.index_copy_(0, torch.as_tensor(slots, device=local.device),
                             allb[q * cmax:q * cmax + counts[q]])
    return full


def block_qr_distributed(a, cfg: BlockConfig, rng: RngState, *, group=None, engine=None, sketch="fresh"):
    """``block_qr(a, cfg, rng)`` (blocked.py:175) with the columns spread over the
    ranks of ``group``; every rank passes the same ``a`` and gets (R, perm) back.
    R is upper trapezoidal (m x n, numpy), perm as in ``Factorization.perm``."""
    engine = engine if engine is not None else CudaStepEngine()
    d = _Dist(group)
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape
    full, _ = engine.alloc(m, n)
    full[:n, :m].copy_(engine.torch.from_numpy(np.ascontiguousarray(a.T)))
    a_loc, lda = scatter_columns(full, m, n, cfg.block, d.world, d.rank, engine)
    del full
    res = factorize_local(a_loc, lda, m, n, cfg, rng, group=group, engine=engine, sketch=sketch)
    r_full = gather_r(res, engine, group)
    r = np.asfortranarray(r_full[:n, :m].cpu().numpy().T)
    return np.triu(r), res.perm

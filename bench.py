"""Benchmark: HQRRP (block_qr, BASELINE.json cfg 3) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one full block_qr factorization of an n x n i.i.d. N(0,1) fp64
matrix (cfg 3: n=10000, b=256, p=16, q=0) starting from a pristine copy of A
already resident in HBM (the copy is part of the step, as blocked.py:161
copies its input).  Headline sketch mode: HQRRP's downdated sketch (G drawn
once from RngState(1), Y = G A, Y2 <- Y2 - G1 R12 per panel; SURVEY section 8
"the mode used for the throughput numbers"); the reference's fresh per-panel
sketch (reference semantics, +2 m' n' (b+p) flops per panel that the 4/3 n^3
count does not credit) is timed on the same input and reported as `variant`.
Metric: fp64 TFLOP/s on the (4/3) n^3 count.

* value: device time (CUDA events on the library stream), max over ranks.
* e2e: the public C ABI entry rq_factorize_host from pinned host memory,
  H2D of A and D2H of R + perm inside the timed region.
* roofline: the trailing-update DMMA GEMMs (the dominant kernel class),
  algorithmic flops 4 m' b n2 + 3 b^2 n2 per panel over
  their CUDA-event time in the timed steps, against the measured FP64 DMMA
  peak (profiles/probe_r01.jsonl; MEASURED_PEAKS.json has no FP64 entry).
* cpu_baseline / --impl reference: the CPU oracle (oracle/, a restatement of
  the reference's numba/numpy path; the reference is pure Python, so there is
  nothing to compile) on this host's cores, over a bounded sample: the first
  `--ref-panels` panels of the same factorization, credited with their share
  of the 4/3 n^3 count (sum of 4 m' b n2 over the sampled panels).
N > 1 (torchrun, one rank per GPU, NCCL): the 1-D block-cyclic driver
(paper_1505_08115_b200/dist.py) factors ONE n x n matrix spread
over the ranks (strong scaling: value = whole-job (4/3) n^3 / max-over-ranks
device time).  `--dist` runs that driver at N = 1 as well.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 36.96  # measured DMMA m16n8k4 peak on this pool's B200 (profiles/probe_r01.jsonl)
TF32X3_PEAK_TFLOPS = 1100.0 / 3  # nominal dense TF32 / 3 split products (B200_PROFILING.md; not measured)
CATS = ["trailing_gemm", "other_gemm", "sketch_cpqr", "panel_leaf", "other", "small_cpqr", "sketch_gemm",
        "panel_gemm", "tfactor", "moves", "copy2d", "rng", "splitk_reduce"]
BW_CATS = {"moves": 9, "copy2d": 10, "rng": 11, "splitk_reduce": 12}


def hbm_peak():
    """Measured HBM copy bandwidth (MEASURED_PEAKS.json, driver-written), else the recipe's fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy, read+write)"
    except Exception:
        return 7700.0, "B200 nominal 7.7 TB/s (B200_PROFILING.md fallback)"


def read_breakdown(lib, handle, check):
    """Per-class device time of one profiled step, plus algorithmic GB/s for the bandwidth classes."""
    cats = {}
    peak, src = hbm_peak()
    for c, name in enumerate(CATS):
        t, f, k = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
        check(lib.rq_profile_read(handle, c, ctypes.byref(t), ctypes.byref(f), ctypes.byref(k)))
        cats[name] = {"ms": t.value, "launches": k.value}
        if name in BW_CATS:
            by = ctypes.c_double()
            check(lib.rq_profile_bytes(handle, c, ctypes.byref(by)))
            gbs = by.value / (t.value * 1e-3) / 1e9 if t.value > 0 else None
            cats[name].update({"bytes": by.value, "gbs": gbs, "frac_of_hbm": (gbs / peak) if gbs else None})
    cats["hbm_peak_gbs"] = {"value": peak, "source": src}
    return cats
METRIC = "fp64 TFLOP/s (4/3·n³ count) for HQRRP at n=10k–40k; % of FP64 TC peak"


def nominal_panel_flops(m, n, b, panels=None):
    """4 m' b n2 per non-final panel: sums to ~(4/3) n^3 for square A."""
    tot, s, k = 0.0, 0, 0
    while n - s > b and (panels is None or k < panels):
        mp, n2 = m - s, n - s - b
        tot += 4.0 * mp * b * n2
        s += b
        k += 1
    return tot


def trailing_algorithmic_flops(m, n, b):
    tot, s = 0.0, 0
    while n - s > b:
        mp, n2 = m - s, n - s - b
        tot += 4.0 * mp * b * n2 + 3.0 * b * b * n2
        s += b
    return tot


class Clocks:
    """nvidia-smi sampling during the timed region."""

    def __init__(self, idx):
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{idx}.csv")
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(idx),
                 "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        self.wait_ready()

    def wait_ready(self, timeout=8.0):
        """Block until the sampler has written its first line: nvidia-smi's start-up (NVML init,
        device enumeration) perturbs a running GPU for tens of ms, so it must be over before the
        timed region starts; the steady 200 ms polling that follows is what the recipe asks for."""
        if self.proc is None:
            return
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < timeout:
            try:
                if os.path.getsize(self.path) > 0:
                    return
            except OSError:
                pass
            if self.proc.poll() is not None:
                return
            time.sleep(0.05)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() in ("active", "1"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_oracle_sample(n, b, p, panels, threads=None):
    """Time the CPU oracle on the first `panels` panels of the cfg-3 factorization."""
    from oracle import randqr_oracle as O

    a = O.gaussian_matrix(n, n, O.RngState(0))
    cfg = O.BlockConfig(b, O.SketchConfig(b, p, 0))
    t0 = time.perf_counter()
    O.block_qr(a, cfg, O.RngState(1), max_panels=panels)
    dt = time.perf_counter() - t0
    return nominal_panel_flops(n, n, b, panels) / dt / 1e12, dt


def cpu_oracle_full(n, b, p):
    """One complete oracle factorization (fresh sketch) of an n x n N(0,1) matrix: (seconds, TFLOP/s)."""
    from oracle import randqr_oracle as O

    a = O.gaussian_matrix(n, n, O.RngState(0))
    cfg = O.BlockConfig(b, O.SketchConfig(b, p, 0))
    t0 = time.perf_counter()
    O.block_qr(a, cfg, O.RngState(1))
    dt = time.perf_counter() - t0
    return dt, 4.0 / 3.0 * n ** 3 / dt / 1e12


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU path (oracle restatement) on host cores."""
    if rank != 0:
        return
    from oracle import randqr_oracle as O

    n, b, p = args.n, args.b, args.p
    a = O.gaussian_matrix(n, n, O.RngState(0))
    cfg = O.BlockConfig(b, O.SketchConfig(b, p, 0))
    for _ in range(args.warmup):
        O.block_qr(a, cfg, O.RngState(1), max_panels=args.ref_panels)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.block_qr(a, cfg, O.RngState(1), max_panels=args.ref_panels)
    dt = time.perf_counter() - t0
    flops = nominal_panel_flops(n, n, b, args.ref_panels) * args.steps
    val = flops / dt / 1e12
    cores = host_cores()
    line = {
        "metric": METRIC, "value": val, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": f"cfg3 HQRRP fp64 n={n} b={b} p={p} q=0, fresh sketch; "
                               f"bounded sample: first {args.ref_panels} panel(s) per step",
                   "n": n, "b": b, "p": p},
        "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": cores, "kind": "port",
                         "sample": f"first {args.ref_panels} panel(s) of n={n}, credited 4 m' b n2 per panel"},
        "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def device_time_n(eng, lib, check, torch, stream, n, b, p, mode, pk, steps=None, flags=0):
    """One n x n factorization per step on the device (A resident, pristine copy per step)."""
    import paper_1505_08115_b200 as rq
    from paper_1505_08115_b200 import _lib

    steps = steps or (2 if n <= 20000 else 1)
    with torch.cuda.stream(stream):
        a0, ld = rq.gaussian_matrix_device(n, n, rq.RngState(0), engine=eng)
        work = torch.empty_like(a0)
        perm = torch.empty(n, dtype=torch.int64, device=eng.device)
    cfg = _lib.rq_config(b, p, 0, -1, pk, 0, mode, flags)

    def step():
        with torch.cuda.stream(stream):
            work.copy_(a0)
        ctr = ctypes.c_uint64(0)
        check(lib.rq_factorize(eng.handle, ctypes.byref(cfg), n, n, ctypes.c_void_p(work.data_ptr()), ld,
                               ctypes.c_uint64(1), ctypes.byref(ctr), ctypes.c_void_p(perm.data_ptr())))

    step()
    torch.cuda.synchronize()
    clocks = Clocks(eng.device.index)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / steps
    clk = clocks.stop()
    tf = 4.0 / 3.0 * n ** 3 / (ms * 1e-3) / 1e12
    del a0, work, perm
    torch.cuda.empty_cache()
    return {"ms_per_step": ms, "value": tf, "unit": "TFLOP/s",
            "fraction_of_fp64_peak": tf / FP64_PEAK_TFLOPS if not flags else None,
            "steps": steps, "warmup": 1, "sm_mhz": clk.get("sm_mhz"), "reasons": clk.get("reasons")}


def trailing_flops_rank(m, n, b, world, rank):
    """Algorithmic trailing-update flops of one rank's columns (block-cyclic)."""
    from paper_1505_08115_b200.dist import BlockCyclic

    lay = BlockCyclic(n, b, world)
    tot, s, i = 0.0, 0, 0
    while n - s > b:
        mp = m - s
        n2 = lay.n_local(rank) - lay.local_from(rank, i + 1)
        tot += 4.0 * mp * b * n2 + 3.0 * b * b * n2
        s += b
        i += 1
    return tot


def run_distributed(args, dist, rank, world, local):
    """One n x n factorization spread over `world` GPUs (dist.py), timed on the device."""
    import torch

    import paper_1505_08115_b200 as rq
    from paper_1505_08115_b200 import dist as rqd
    from paper_1505_08115_b200.errors import check

    n, b, p = args.n, args.b, args.p
    m = n
    stream = torch.cuda.Stream()
    eng = rq.Engine(local, stream=stream)
    se = rqd.CudaStepEngine(eng)
    cfg = rq.BlockConfig(b, rq.SketchConfig(b, p, 0))
    with torch.cuda.stream(stream):
        a_full, _ = rq.gaussian_matrix_device(m, n, rq.RngState(0), engine=eng)
        a0_loc, lda = rqd.scatter_columns(a_full, m, n, b, world, rank, se)
        del a_full
        work = torch.empty_like(a0_loc)
    nloc = rqd.BlockCyclic(n, b, world).n_local(rank)

    def step():
        with torch.cuda.stream(stream):
            work.copy_(a0_loc)
            rqd.factorize_local(work, lda, m, n, cfg, rq.RngState(1), engine=se, sketch=args.sketch)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    time.sleep(0.3)
    launches0 = eng.launches
    dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    ms = ev0.elapsed_time(ev1)
    launches = eng.launches - launches0
    clk = clocks.stop()
    check(eng.lib.rq_set_profiling(eng.handle, 1))  # breakdown from one separate profiled step
    step()
    torch.cuda.synchronize()
    cats = read_breakdown(eng.lib, eng.handle, check)
    check(eng.lib.rq_set_profiling(eng.handle, 0))
    tt = torch.tensor([ms], device=eng.device, dtype=torch.float64)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms_max = float(tt.item())
    flops_step = 4.0 / 3.0 * n ** 3
    value = args.steps * flops_step / (ms_max * 1e-3) / 1e12
    t_trail = cats["trailing_gemm"]["ms"]
    achieved = trailing_flops_rank(m, n, b, world, rank) / (t_trail * 1e-3) / 1e12 if t_trail > 0 else None

    e2e = None
    if not args.no_e2e:
        # host (pinned) local columns -> device -> factorize -> local R columns back to the host
        ha = torch.empty_like(a0_loc, device="cpu").pin_memory()
        ha.copy_(a0_loc.cpu())
        hr = torch.empty_like(ha).pin_memory()

        def e2e_step():
            with torch.cuda.stream(stream):
                work.copy_(ha, non_blocking=True)
                rqd.factorize_local(work, lda, m, n, cfg, rq.RngState(1), engine=se, sketch=args.sketch)
                hr.copy_(work, non_blocking=True)
            stream.synchronize()

        e2e_step()
        dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        k_e2e = max(1, min(args.steps, 3))
        for _ in range(k_e2e):
            e2e_step()
        ev1.record(stream)
        torch.cuda.synchronize()
        dt = ev0.elapsed_time(ev1) * 1e-3
        tt = torch.tensor([dt], device=eng.device, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
        e2e = {"value": k_e2e * flops_step / dt / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": m * n * 8, "d2h_bytes_per_step": m * n * 8,
               "note": "per rank: its block-cyclic columns in and its R columns out (summed over ranks)"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"cfg3 HQRRP fp64 n={n} b={b} p={p} q=0, {args.sketch} sketch, "
                                   f"1-D block-cyclic columns over {world} GPU(s)",
                       "n": n, "b": b, "p": p, "q": 0, "sketch": args.sketch, "method": "m1", "matrix": "gauss",
                       "parallelism": f"block-cyclic columns x{world} (NCCL all-gather / send-recv / broadcast)",
                       "l2": "inputs (800 MB) larger than L2 (126 MB)"},
            "fraction_of_fp64_peak": value / (FP64_PEAK_TFLOPS * world),
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": (achieved / FP64_PEAK_TFLOPS) if achieved else None, "traffic": None,
                         "kernel": "gemm_f64_kernel (rank 0's trailing updates, rq_panel_apply)",
                         "peak_source": "measured DMMA peak, profiles/probe_r01.jsonl"},
            "breakdown_ms_per_step": cats,
            "local_columns_rank0": nloc,
            "clocks": clk,
            "gpu_launches": launches,
            "e2e": e2e,
            "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def run_fp32(args, local):
    """cfg 3 fp32: one factorization per step on one GPU (fp32.py), device-timed."""
    import torch

    import paper_1505_08115_b200 as rq
    from paper_1505_08115_b200 import dist as rqd
    from paper_1505_08115_b200.fp32 import Fp32StepEngine

    torch.cuda.set_device(local)
    n, b, p = args.n, args.b, args.p
    m = n
    stream = torch.cuda.Stream()
    eng = rq.Engine(local, stream=stream)
    se = Fp32StepEngine(eng)
    cfg = rq.BlockConfig(b, rq.SketchConfig(b, p, 0))
    with torch.cuda.stream(stream):
        a64, _ = rq.gaussian_matrix_device(m, n, rq.RngState(0), engine=eng)
        a0, lda = se.alloc(m, n)
        a0[:n, :m] = a64[:n, :m]
        del a64
        work = torch.empty_like(a0)

    def step():
        with torch.cuda.stream(stream):
            work.copy_(a0)
            rqd.factorize_local(work, lda, m, n, cfg, rq.RngState(1), engine=se, sketch=args.sketch)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    time.sleep(0.3)
    launches0 = eng.launches
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    clk = clocks.stop()
    flops_step = 4.0 / 3.0 * n ** 3
    value = args.steps * flops_step / (ms * 1e-3) / 1e12
    line = {
        "metric": "fp32 TFLOP/s (4/3·n³ count) for HQRRP, cfg 3 fp32 variant", "value": value, "unit": "TFLOP/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32 (GEMMs) / f64 (serial kernels)",
        "data": "synthetic",
        "config": {"workload": f"cfg3 fp32 HQRRP n={n} b={b} p={p} q=0, {args.sketch} sketch", "n": n, "b": b, "p": p,
                   "sketch": args.sketch,
                   "parallelism": "single", "l2": "inputs (400 MB) larger than L2 (126 MB)"},
        "note": "fp32 storage; sketch and trailing GEMMs = this library's tcgen05 3xTF32 GEMM (rq_gemm_f32, "
                "TMA + TMEM); sketch CPQR, panel QR, b x b CPQR, T in this library's fp64 kernels; panel-step "
                "driver (dist.factorize_local, world size 1) (fp32.py)",
        "clocks": clk, "gpu_launches": eng.launches - launches0, "e2e": None, "cpu_baseline": None,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=10000)
    ap.add_argument("--b", type=int, default=256)
    ap.add_argument("--p", type=int, default=16)
    ap.add_argument("--ref-panels", type=int, default=1)
    ap.add_argument("--cpu-panels", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--sketch", default="downdate", choices=["fresh", "downdate"],
                    help="headline sketch mode: downdate = HQRRP (Y = G A once, Y2 <- Y2 - G1 R12 per panel, "
                         "the north star's hot path); fresh = the reference's per-panel fresh sketch")
    ap.add_argument("--no-variant", action="store_true", help="skip timing the other sketch mode")
    ap.add_argument("--per-n", default="20000,40000",
                    help="extra sizes timed on the device in the same run (reported under per_n; '' = none)")
    ap.add_argument("--method", default="m1", choices=["m1", "m2", "m3"],
                    help="m1 block_qr permutation pivots (headline), m2 reflector pivots, m3 block_rrqr")
    ap.add_argument("--q", type=int, default=0, help="power iterations of the sketch")
    ap.add_argument("--dist", action="store_true", help="use the block-cyclic multi-GPU driver even at N = 1")
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"],
                    help="f32: cfg 3's fp32 variant -- the monolithic driver with the trailing-update GEMMs as "
                         "tcgen05 3xTF32 products (RQ_FLAG_TF32_UPDATE); --f32-steps: fp32 storage through the "
                         "panel-step driver (fp32.py)")
    ap.add_argument("--f32-steps", action="store_true")
    ap.add_argument("--matrix", default="gauss", choices=["gauss", "cfg4"],
                    help="gauss: N(0,1) (cfg 3); cfg4: U diag(max(10^(-12j/2000),1e-15)) V^T")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.dtype == "f32" and args.f32_steps:
        run_fp32(args, local)
        return

    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1 or args.dist:
        import torch.distributed as dist

        for k, v in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29517"), ("RANK", "0"), ("WORLD_SIZE", "1")):
            os.environ.setdefault(k, v)

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        if args.method == "m1" and args.q == 0 and args.matrix == "gauss":
            return run_distributed(args, dist, rank, world, local)
        if rank == 0:
            print(json.dumps({"metric": METRIC, "unavailable": "multi-GPU runs cover m1 fresh q=0 (dist.py)"}))
        dist.destroy_process_group()
        return

    import paper_1505_08115_b200 as rq
    from paper_1505_08115_b200 import _lib
    from paper_1505_08115_b200.errors import check

    n, b, p = args.n, args.b, args.p
    m = n
    stream = torch.cuda.Stream()
    eng = rq.Engine(local, stream=stream)
    lib = eng.lib
    # A = gaussian_matrix(n, n, RngState(0)): same counter-based stream as the reference
    with torch.cuda.stream(stream):
        a0, ld = rq.gaussian_matrix_device(m, n, rq.RngState(0), engine=eng)
        if args.matrix == "cfg4":
            # cfg 4: U diag(s) V^T, U and V = haar_orthonormal(n, RngState(0))
            # drawn U first (matrices.py:34-41, 67-68), s_j = max(10^(-12 j / 2000), 1e-15); built on
            # the device with this library's unpivoted QR, outside the timed region
            from paper_1505_08115_b200.matrices import haar_orthonormal_device

            hr = rq.RngState(0)
            u, _ = haar_orthonormal_device(n, hr, engine=eng)
            v, _ = haar_orthonormal_device(n, hr, engine=eng)
            jj = torch.arange(1, n + 1, device=eng.device, dtype=torch.float64)
            sv = torch.clamp(10.0 ** (-12.0 * jj / 2000.0), min=1e-15)
            a0[:n, :n] = v[:n, :n].T @ (u[:n, :n] * sv[:, None])  # storage = A^T = V diag(s) U^T
            del u, v
        work, _ = eng.alloc_matrix(m, n)
        perm = torch.empty(n, dtype=torch.int64, device=eng.device)
    if args.method != "m1":
        args.sketch = "fresh"  # reflector pivots / block_rrqr: the reference's fresh sketches only
    mode = _lib.RQ_SKETCH_FRESH if args.sketch == "fresh" else _lib.RQ_SKETCH_DOWNDATE
    pk = _lib.RQ_PIVOT_PERMUTATION if args.method == "m1" else _lib.RQ_PIVOT_REFLECTORS
    f32 = args.dtype == "f32"
    cfg = _lib.rq_config(b, p, args.q, -1, pk, 1 if args.method == "m3" else 0, mode,
                         _lib.RQ_FLAG_TF32_UPDATE if f32 else 0)
    if args.method != "m1":
        args.no_variant = True  # the downdated sketch applies to permutation pivots only

    def step():
        with torch.cuda.stream(stream):
            work.copy_(a0)
        ctr = ctypes.c_uint64(0)
        check(lib.rq_factorize(eng.handle, ctypes.byref(cfg), m, n, ctypes.c_void_p(work.data_ptr()), ld,
                               ctypes.c_uint64(1), ctypes.byref(ctr), ctypes.c_void_p(perm.data_ptr())))

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    time.sleep(0.3)
    launches0 = eng.launches
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    h0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    host_ms = (time.perf_counter() - h0) * 1e3 / args.steps  # enqueue time (rq_factorize is enqueue-only)
    ev1.record(stream)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    launches = eng.launches - launches0
    clk = clocks.stop()
    # per-class breakdown: a separate profiled step (CUDA events around every launch cost ~5%,
    # so the timed region above runs without them)
    check(lib.rq_set_profiling(eng.handle, 1))
    step()
    torch.cuda.synchronize()
    cats = read_breakdown(lib, eng.handle, check)
    check(lib.rq_set_profiling(eng.handle, 0))
    ms_max = ms
    if dist is not None:
        tt = torch.tensor([ms], device=eng.device, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_max = float(tt.item())
    flops_step = 4.0 / 3.0 * n ** 3
    value = world * args.steps * flops_step / (ms_max * 1e-3) / 1e12

    # the other sketch mode, same workload (reported beside the headline)
    variant = None
    if not args.no_variant:
        other = "downdate" if args.sketch == "fresh" else "fresh"
        cfg.sketch_mode = _lib.RQ_SKETCH_DOWNDATE if other == "downdate" else _lib.RQ_SKETCH_FRESH
        for _ in range(2):
            step()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        vms = ev0.elapsed_time(ev1) / args.steps
        variant = {"sketch": other, "value": flops_step / (vms * 1e-3) / 1e12, "ms_per_step": vms}
        cfg.sketch_mode = mode

    # device-time sub-results at the north star's larger sizes (cfg 5 family), same mode and timer
    per_n = None
    if args.per_n and args.method == "m1" and args.matrix == "gauss" and world == 1:
        per_n = {}
        for n_big in [int(x) for x in args.per_n.split(",") if x]:
            per_n[str(n_big)] = device_time_n(eng, lib, check, torch, stream, n_big, b, p, mode, pk,
                                              flags=cfg.flags)
        torch.cuda.synchronize()

    # dominant kernel roofline: the trailing-update DMMA GEMMs
    t_trail = cats["trailing_gemm"]["ms"]
    achieved = trailing_algorithmic_flops(m, n, b) / (t_trail * 1e-3) / 1e12 if t_trail > 0 else None

    # e2e through the public C ABI with pinned host buffers
    e2e = None
    if not args.no_e2e:
        ha = torch.empty((n, ld), dtype=torch.float64, pin_memory=True)
        ha.copy_(a0.cpu())
        hr = torch.empty((n, ld), dtype=torch.float64, pin_memory=True)
        hp = torch.empty(n, dtype=torch.int64, pin_memory=True)

        def e2e_step():
            ctr = ctypes.c_uint64(0)
            check(lib.rq_factorize_host(eng.handle, ctypes.byref(cfg), m, n, ctypes.c_void_p(ha.data_ptr()), ld,
                                        ctypes.c_uint64(1), ctypes.byref(ctr), ctypes.c_void_p(hr.data_ptr()), ld,
                                        ctypes.c_void_p(hp.data_ptr())))

        e2e_step()
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        k_e2e = max(1, min(args.steps, 3))
        for _ in range(k_e2e):
            e2e_step()
        dt = time.perf_counter() - t0
        if dist is not None:
            tt = torch.tensor([dt], device=eng.device, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = float(tt.item())
        e2e = {"value": world * k_e2e * flops_step / dt / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": m * n * 8, "d2h_bytes_per_step": m * n * 8 + n * 8}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        val, dt = cpu_oracle_sample(n, b, p, args.cpu_panels)
        full = []
        for (fn_, fb_, fp_) in ((2000, 64, 10), (4000, 128, 10)):
            sec, tf = cpu_oracle_full(fn_, fb_, fp_)
            full.append({"n": fn_, "b": fb_, "p": fp_, "seconds": sec, "value": tf, "unit": "TFLOP/s"})
        cpu = {"value": val, "unit": "TFLOP/s", "cores": host_cores(), "kind": "port",
               "sample": f"PORT (oracle/: restatement of the reference's numba sweeps + OpenBLAS GEMMs, fresh "
                         f"sketch), PANEL SAMPLE: the first {args.cpu_panels} panels of the n={n} factorization "
                         f"({dt:.1f} s), EXTRAPOLATED: rate = those panels' 4 m' b n2 credit / their time",
               "full_factorizations": full,
               "full_note": "complete oracle block_qr runs (N(0,1), seed 0 / sketch seed 1) timed in the same run"}

    if rank == 0:
        line = {
            "metric": METRIC if not f32 else "fp32 TFLOP/s (4/3·n³ count) for HQRRP, cfg 3 fp32 variant",
            "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "f64" if not f32 else "f32 (trailing-update GEMMs: tcgen05 3xTF32, fp32 accumulation; "
                                          "panels / sketch / pivots fp64)",
            "data": "synthetic",
            "config": {"workload": (f"cfg3 HQRRP fp64 n={n} b={b} p={p} q={args.q}, {args.sketch} sketch"
                                    + (" (reference semantics)" if args.sketch == "fresh" else " (HQRRP downdate)"))
                                   if args.method == "m1" else
                                   f"{args.method} ({'block_rrqr' if args.method == 'm3' else 'reflector pivots'}) "
                                   f"fp64 n={n} b={b} p={p} q={args.q}, matrix={args.matrix}",
                       "n": n, "b": b, "p": p, "q": args.q, "sketch": args.sketch, "method": args.method,
                       "matrix": args.matrix,
                       "parallelism": "replicas" if world > 1 else "single",
                       "l2": "inputs (800 MB) larger than L2 (126 MB)"},
            "fraction_of_fp64_peak": value / FP64_PEAK_TFLOPS if not f32 else None,
            "roofline": ({"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                          "frac": (achieved / FP64_PEAK_TFLOPS) if achieved else None,
                          # ncu --set full, one A2 -= V W2 launch (n = 10000, K = b = 256):
                          # dram read + write vs 1.640e9 algorithmic bytes (profiles/ncu_gemm_nn_r01.txt)
                          "traffic": 1.6466e9 if n == 10000 and b == 256 else None,
                          "traffic_note": "bytes per launch of A2 -= V W2 at panel 1; algorithmic 1.640e9",
                          "kernel": "gemm_f64_kernel (trailing update: V^T A2, T^T W, A2 -= V W2, Q2^T top)",
                          "peak_source": "measured DMMA peak, profiles/probe_r01.jsonl"} if not f32 else
                         {"bound": "tensor", "achieved": achieved, "peak": TF32X3_PEAK_TFLOPS, "unit": "TFLOP/s",
                          "frac": (achieved / TF32X3_PEAK_TFLOPS) if achieved else None, "traffic": None,
                          "kernel": "gemm_tf32x3_kernel<double> (trailing update on tcgen05, 3 TF32 products "
                                    "per 2MNK flop)",
                          "peak_source": "B200 nominal dense TF32 1.1 PFLOP/s (B200_PROFILING.md) / 3 products; "
                                         "MEASURED_PEAKS.json has no TF32 entry"}),
            "breakdown_ms_per_step": cats,
            "breakdown_note": "one separate profiled step (CUDA events per launch); classes overlap in time "
                              "(W = V^T A2 and T run beside the b x b CPQR)",
            "variant": variant,
            "per_n": per_n,
            "clocks": clk,
            "gpu_launches": launches,
            "host_enqueue_ms_per_step": host_ms,
            "host_enqueue_note": "host time of the rq_factorize calls in the timed loop (they only enqueue; "
                                 "below ms_per_step = the GPU never waits on the host)",
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

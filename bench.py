#!/usr/bin/env python
"""Benchmark of the hot path: H X (+ halo), S = X^T (H X) (+ cross-rank reduction), X C.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--impl ours|reference]

Workload: BASELINE.json configs[4], the weak-scaling config at G = N GPUs
(64 x 64 x 64N cells, Q4, M = 512N orbitals, r = 8 cells, sigma = 2 cells;
synthetic seeded inputs).  --config q2|q4|proj|smoke|weakG
selects another BASELINE config (single-GPU parity/perf lines).

One step = CellOperator.apply(H, X, HX) -> tmmult(X, HX, S) -> mmult(X, C, XC)
through the drop-in API.  Inputs stay resident in HBM for `value`; `e2e`
adds, every step, the H2D copy of X's structural nonzeros from pinned host
memory (upload_support_values) and the D2H read of S.  Inputs exceed L2 (X alone is 2.6 GB stored at G = 1), so no L2 flush is needed.

Metric unit: algorithmic GFlop/s, F = pairs * (24 n^4 + 8 n^3) for H X
(the implemented collocation count, < the reference 36 n^4 + 8 n^3;
SURVEY 8(d): F = min(reference, implemented)) + 2 sum_rows kX kZ (S) +
2 sum_rows kX^2 (X C), identical for both arms.

--impl reference times the reference algorithm's C restatement
(oracle/cellop.c: Algorithm 6 on the BCSR layout, all lanes, 18
contractions; tmmult / mmult block loops) on the host cores, rank 0 only,
on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


# -- clocks -----------------------------------------------------------------------


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.rows = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx.append(float(r[2]))
                for k, name in enumerate(names):
                    if r[5 + k].lower().startswith("active"):
                        reasons.add(name)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# -- workload accounting ---------------------------------------------------------------


def workload_counts(st):
    """Algorithmic work of one step on this rank."""
    from scipy import sparse

    op, x, layout = st.op, st.x, st.layout
    n = st.prob.cfg.degree + 1
    xmask = x.support.local_mask(layout).astype(np.int32)
    a_cell = op.cell_local_rows_matrix(xmask.shape[0])
    act = (a_cell @ xmask).tocsr()
    act.data[:] = 1
    hxmask = (a_cell.T @ act).tocsr()
    hxmask.data[:] = 1
    own = layout.owned_rows[1] - layout.owned_rows[0]
    kx = np.diff(xmask.indptr)[:own].astype(np.int64)
    kz = np.diff(hxmask.indptr)[:own].astype(np.int64)
    pairs = int(act.nnz)
    f_ref = 36 * n**4 + 8 * n**3
    f_imp = 24 * n**4 + 8 * n**3
    cells = len(op.cells)
    return {
        "pairs": pairs,
        "nnzX": int(kx.sum()),
        "nnzHX": int(kz.sum()),
        "cells": cells,
        "flops_hx": pairs * min(f_ref, f_imp),
        "flops_hx_reference_formulation": pairs * f_ref,
        "flops_s": int(2 * np.sum(kx * kz)),
        "flops_xc": int(2 * np.sum(kx * kx)),
        "bytes_hx": int(8 * kx.sum() + 8 * kz.sum() + cells * (8 * n**3 + 4 * n**3) + 4 * pairs),
        "bytes_s": int(8 * (kx.sum() + kz.sum())),
        "bytes_xc": int(8 * 2 * kx.sum()),
    }


def measure_fp64_peak(torch, lib, C, dev):
    """FP64 throughput of this GPU, TFLOP/s: (DFMA probe, DMMA probe).  The K1
    roofline denominator is the larger of the two (MEASURED_PEAKS.json has no
    FP64 entry)."""
    from paper_1907_01005_b200 import _lib

    scratch = torch.zeros(8, dtype=torch.float64, device=dev)
    sm = C.c_int()
    lib.bmv_device_sm_count(C.byref(sm))
    blocks = sm.value * 8
    flops = C.c_double()
    st = _lib.stream_handle(dev)
    out = []
    for fn, iters in ((lib.bmv_fp64_peak_kernel, 2048), (lib.bmv_fp64_dmma_peak_kernel, 1024)):
        for _ in range(2):
            _lib.check(fn(_lib.dptr(scratch), blocks, 64, C.byref(flops), st))
        torch.cuda.synchronize()
        best = 0.0
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _lib.check(fn(_lib.dptr(scratch), blocks, iters, C.byref(flops), st))
            e1.record()
            e1.synchronize()
            best = max(best, flops.value / (e0.elapsed_time(e1) * 1e-3) / 1e12)
        out.append(best)
    return tuple(out)


def peaks_file():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except ValueError:
            return {}
    return {}


# -- the CPU reference arm -----------------------------------------------------------------


def bench_config(name, prob, st):
    """The `config` object of both arms' JSON lines (same workload, same text)."""
    return {"workload": name, "note": prob.cfg.note,
            "step": "apply H (halo) + tmmult S=X^T(HX) (compress) + mmult XC",
            "storage": "slab layout (slabs.py): X %.3f GB, H X %.3f GB, X C %.3f GB" % (
                st.x.slab.off[-1] * 8e-9, st.hx.slab.off[-1] * 8e-9, st.xc.slab.off[-1] * 8e-9),
            "l2": "inputs larger than L2 (126 MB): no flush between steps"}


def reference_arm(args, rank, world):
    """The reference algorithm on the host cores: the C restatement of the
    reference loops (oracle/cellop.c: Algorithm 6 on the reference BCSR layout,
    all lanes, 18 contractions; tmmult / mmult block loops), inputs built with
    the package's numpy setup path only (BMV_PLAN_NATIVE=0: no repo library is
    loaded by this process besides oracle/liboracle.so)."""
    os.environ["BMV_PLAN_NATIVE"] = "0"
    if rank != 0:
        return
    import torch  # noqa: F401  (matrices on the CPU)

    from oracle import c_oracle as CO
    from paper_1907_01005_b200 import problem as P
    from paper_1907_01005_b200.comm import serial_context

    name = args.config or f"weak{world}"
    prob = P.build_problem(name, world)
    st = P.make_rank_setup(serial_context("cpu"), prob, device="cpu", projection=True)
    cnt = workload_counts(st)
    f_total = cnt["flops_hx"] + cnt["flops_s"] + cnt["flops_xc"]
    threads = os.cpu_count() or 1
    op = st.op
    deg = prob.cfg.degree
    n_cells = len(op.cells)
    x = CO.reference_values(st.x)
    c_vals = CO.reference_values(st.c)
    vq_cache = {}

    def hx_cells(k):
        if k not in vq_cache:
            vq_cache.clear()
            vq_cache[k] = CO.potential_gaussian(prob.potential, op.cell_origins[:k], deg,
                                                prob.mesh.spacing, threads)
        h = CO.reference_zeros(st.hx)
        t0 = time.perf_counter()
        CO.cellop_apply(deg, prob.mesh.spacing, "h", op._lb[:k], op._rib[:k], op.cell_color[:k],
                        vq_cache[k], CO.matrix_meta(st.x), CO.matrix_meta(st.hx), st.x.col_strides,
                        st.x.col_blocks.sizes, x, h, threads=threads)
        return time.perf_counter() - t0, h

    holder = {}

    def products():
        h_full = holder["h"]  # H X of the sampled cells (the loops' work is value-independent)
        t0 = time.perf_counter()
        CO.tmmult(st.x, st.hx, st.s, x, h_full, threads=threads)
        CO.mmult(st.x, st.c, st.xc, x, c_vals, threads=threads)
        return time.perf_counter() - t0

    # sample size: about 2 s of H X per step on this host
    probe = max(1, min(n_cells, 256))
    t_probe, holder["h"] = hx_cells(probe)
    k = int(min(n_cells, max(probe, probe * 2.0 / max(t_probe, 1e-6))))
    frac = k / max(n_cells, 1)
    for _ in range(args.warmup):
        _, holder["h"] = hx_cells(k)
        products()
    times = []
    for _ in range(args.steps):
        t_h, holder["h"] = hx_cells(k)
        times.append(t_h / frac + products())
    t_step = float(np.mean(times))  # H X extrapolated by cells + S and X C timed in full
    value = f_total / t_step / 1e9
    line = {
        "metric": "matrix-free sparse SpMM fp64 GFlop/s (algorithmic) at N B200",
        "impl": "reference", "value": round(value, 3), "unit": "GFlop/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_step * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded splitmix64 fill, Gaussian potential; SURVEY 0.1)",
        "config": bench_config(name, prob, st),
        "cpu_baseline": {"value": round(value, 3), "unit": "GFlop/s", "cores": threads,
                         "kind": "port",
                         "sample": f"H X over the first {k} of {n_cells} Hilbert-ordered cells "
                                   f"({frac:.3f} of the workload, time extrapolated by cells) + "
                                   f"S = X^T (H X) and X C on the whole workload per step; C "
                                   f"restatement of the reference loops (oracle/cellop.c)"},
        "e2e": {"value": round(value, 3), "unit": "GFlop/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# -- our arm ---------------------------------------------------------------------------------


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return reference_arm(args, rank, world)

    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_1907_01005_b200 import _lib
    from paper_1907_01005_b200 import problem as P
    from paper_1907_01005_b200.bcsr import mmult, tmmult
    from paper_1907_01005_b200.comm import DistContext, serial_context

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        ctx = DistContext(device=dev)
    else:
        ctx = serial_context(dev)
    lib = _lib.require_device()
    name = args.config or f"weak{world}"
    t_setup = time.time()
    prob = P.build_problem(name, world)
    st = P.make_rank_setup(ctx, prob, projection=True, device=dev)
    st.c.update_ghost_values()
    spec = prob.spec_h()
    cnt = workload_counts(st)
    # first apply builds the plans (host) and the potential (device)
    st.op.apply(spec, st.x, st.hx)
    torch.cuda.synchronize()
    t_setup = time.time() - t_setup

    launches = {"n": 0}
    plan = st.op.plan_for(st.x, st.hx)

    def step():
        st.op.apply(spec, st.x, st.hx)
        tmmult(st.x, st.hx, st.s)
        mmult(st.x, st.c, st.xc)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = _lib.launch_count()  # counted by libbmv at every kernel launch site
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    gpu_launches = _lib.launch_count() - launches0
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    clk = clocks.stop()

    # per-kernel times (device events; K1 alone = the dominant kernel)
    def timed(fn, reps):
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        b.synchronize()
        return a.elapsed_time(b) / reps

    stream = _lib.stream_handle(dev)

    def k1_only():
        _lib.check(lib.bmv_cellop_apply(plan.handle.raw, 1, *_coef_args(st, spec, dev),
                                        _lib.dptr(st.x.data), _lib.dptr(st.hx.data), 0, stream))

    reps = max(args.steps, 5)
    ms_k1 = max_over_ranks(timed(k1_only, reps))
    ms_apply = max_over_ranks(timed(lambda: st.op.apply(spec, st.x, st.hx), reps))
    ms_tm = max_over_ranks(timed(lambda: tmmult(st.x, st.hx, st.s), reps))
    ms_mm = max_over_ranks(timed(lambda: mmult(st.x, st.c, st.xc), reps))
    st.op.apply(spec, st.x, st.hx)

    f_step = sum_over_ranks(cnt["flops_hx"] + cnt["flops_s"] + cnt["flops_xc"])
    value = f_step / (ms * 1e-3) / 1e9
    peak_dfma, peak_dmma = measure_fp64_peak(torch, lib, C, dev)
    peak_fp64 = max(peak_dfma, peak_dmma)
    k1_tflops = cnt["flops_hx"] / (ms_k1 * 1e-3) / 1e12
    traffic = None
    tp = ROOT / "profiles" / "k1_traffic.json"
    if tp.exists():
        try:
            traffic = json.loads(tp.read_text()).get(name)
        except ValueError:
            traffic = None

    e2e = None
    if not args.no_e2e:
        # inputs arrive from pinned host memory in the compact support format
        # (BlockCsrMatrix.upload_support_values: only the structural nonzeros
        # of X cross PCIe, then a device scatter into the slabs); the
        # step's result S comes back to pinned host memory.  Triple-buffered:
        # the H2D copies of the next steps' X run on a copy stream while step
        # k computes on X buffer k % NB (every step's copy stays inside the
        # timed region; the first copy is not overlapped).
        n_sv = st.x.n_support_values()
        NB = 3
        host_x = [torch.empty(n_sv, dtype=torch.float64, pin_memory=True) for _ in range(NB)]
        for hx_ in host_x:
            hx_.copy_(st.x.download_support_values().cpu())
        host_s = torch.empty(st.s.data.numel(), dtype=torch.float64, pin_memory=True)
        xs = [st.x] + [st.x.copy() for _ in range(NB - 1)]
        dev_x = [torch.empty(n_sv, dtype=torch.float64, device=dev) for _ in range(NB)]
        cstream = torch.cuda.Stream(device=dev)
        copied = [torch.cuda.Event() for _ in range(NB)]
        consumed = [torch.cuda.Event() for _ in range(NB)]
        main = torch.cuda.current_stream(dev)

        def issue_copy(k):
            b = k % NB
            with torch.cuda.stream(cstream):
                cstream.wait_event(consumed[b])
                dev_x[b].copy_(host_x[b], non_blocking=True)
                copied[b].record(cstream)

        def e2e_run(n):
            for b in range(NB):
                consumed[b].record(main)
            for k in range(min(NB - 1, n)):
                issue_copy(k)
            for k in range(n):
                b = k % NB
                main.wait_event(copied[b])
                xk = xs[b]
                xk.upload_support_values(dev_x[b])
                consumed[b].record(main)
                if k + NB - 1 < n:
                    issue_copy(k + NB - 1)
                st.op.apply(spec, xk, st.hx)
                tmmult(xk, st.hx, st.s)
                mmult(xk, st.c, st.xc)
                host_s.copy_(st.s.data, non_blocking=True)

        e2e_run(NB + 1)  # warm-up over every X buffer
        barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        e2e_run(args.steps)
        a1.record()
        a1.synchronize()
        ms_e2e = max_over_ranks(a0.elapsed_time(a1) / args.steps)
        e2e = {"value": round(f_step / (ms_e2e * 1e-3) / 1e9, 3), "unit": "GFlop/s",
               "ms_per_step": round(ms_e2e, 4),
               "h2d_bytes_per_step": int(n_sv * 8),
               "d2h_bytes_per_step": int(host_s.numel() * 8),
               "path": "pinned host -> (copy stream, triple-buffered) device -> "
                       "upload_support_values (compact nnz scatter) -> apply/tmmult/mmult "
                       "-> S to pinned host"}

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu_baseline = cpu_baseline_leg(st, prob, cnt)

    # collective (sum over ranks): every rank computes it
    rk = spmm_roofline(st, cnt, ms_tm, ms_mm, float(peaks_file().get("hbm_gbs", 6650.0)),
                       sum_over_ranks)
    if rank == 0:
        peaks = peaks_file()
        line = {
            "metric": "matrix-free sparse SpMM fp64 GFlop/s (algorithmic) at N B200",
            "value": round(value, 3), "unit": "GFlop/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded splitmix64 fill, Gaussian potential; SURVEY 0.1)",
            "config": bench_config(name, prob, st),
            "dof_vectors_per_s": round(sum_over_ranks(cnt["nnzX"]) / (ms_apply * 1e-3), 1),
            "kernels_ms": {"k1_cellop": round(ms_k1, 4), "apply_total": round(ms_apply, 4),
                           "tmmult": round(ms_tm, 4), "mmult": round(ms_mm, 4)},
            "work": {k: (int(sum_over_ranks(v)) if isinstance(v, int) else v) for k, v in cnt.items()},
            "roofline": {"bound": "fp64", "kernel": "K1 cellop (csrc/bmv_k1.cu, %s<%d>)"
                         % ("k1_plane_kernel" if prob.cfg.degree >= 3 else "k1_pair_kernel",
                            prob.cfg.degree + 1),
                         "achieved": round(k1_tflops, 3), "peak": round(peak_fp64, 3),
                         "unit": "TFLOP/s", "frac": round(k1_tflops / peak_fp64, 4),
                         "frac_vs_dfma": round(k1_tflops / peak_dfma, 4),
                         "peak_source": "measured in-run, max of the DFMA probe (%.2f) and the "
                                        "DMMA probe (%.2f TFLOP/s); MEASURED_PEAKS.json has no "
                                        "FP64 figure" % (peak_dfma, peak_dmma),
                         "hbm_bytes_algorithmic": cnt["bytes_hx"],
                         "hbm_frac_at_k1_time": round(cnt["bytes_hx"] / (ms_k1 * 1e-3) / 1e9
                                                      / float(peaks.get("hbm_gbs", 6650.0)), 4),
                         "traffic": traffic},
            "roofline_kernels": rk,
            "gpu_launches": int(gpu_launches),
            "setup_s": round(t_setup, 1),
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu_baseline,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def spmm_roofline(st, cnt, ms_tm, ms_mm, hbm_gbs, sum_over_ranks):
    """K4 / K5 are HBM-bound.  `achieved` = algorithmic bytes (SURVEY 8(d):
    8 (nnzX + nnzHX) for K4, 16 nnzX for K5) per launch / time; `stored_*`
    gives the same on the slab bytes the kernels actually stream (X + H X
    for K4; X read + X C written for K5)."""
    out = {}
    for name, ms, stored, alg in (
            ("k4_tmmult", ms_tm, 8 * (st.x.n_owned_values + st.hx.n_owned_values),
             cnt["bytes_s"]),
            ("k5_mmult", ms_mm, 8 * (st.x.n_owned_values + st.xc.n_owned_values),
             cnt["bytes_xc"])):
        stored = sum_over_ranks(stored)
        alg = sum_over_ranks(alg)
        gbs = alg / (ms * 1e-3) / 1e9
        out[name] = {"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm_gbs, "unit": "GB/s",
                     "frac": round(gbs / hbm_gbs, 4), "algorithmic_bytes": int(alg),
                     "stored_bytes": int(stored),
                     "stored_frac": round(stored / (ms * 1e-3) / 1e9 / hbm_gbs, 4),
                     "ms": round(ms, 4)}
    return out


def _coef_args(st, spec, dev):
    import ctypes as C

    from paper_1907_01005_b200 import _lib

    coef, stride = st.op.coefficient(spec, dev)
    return (_lib.dptr(coef) if coef is not None else C.c_void_p(None), stride)


def cpu_baseline_leg(st, prob, cnt):
    """C restatement of the reference cell loop on a bounded sample (rank 0, N = 1)."""
    try:
        from oracle import c_oracle as CO
    except Exception as exc:  # pragma: no cover
        return {"value": None, "error": repr(exc)}
    op = st.op
    deg = prob.cfg.degree
    n_cells = len(op.cells)
    threads = os.cpu_count() or 1
    x = CO.reference_values(st.x)
    h = CO.reference_zeros(st.hx)
    xm, hm = CO.matrix_meta(st.x), CO.matrix_meta(st.hx)

    # V at the points from the operator's coefficient (timing only: the parity of
    # the potential is tested in tests/test_gpu_fullsize.py against the numpy oracle)
    coef, stride = op.coefficient(prob.spec_h(), st.x.device)
    w3 = op.kernels.w3.ravel()
    vq_all = coef.view(-1, stride)[:, : w3.size].cpu().numpy() / w3[None, :]

    def run(k):
        vq = vq_all[:k]
        t0 = time.perf_counter()
        CO.cellop_apply(deg, prob.mesh.spacing, "h", op._lb[:k], op._rib[:k], op.cell_color[:k], vq,
                        xm, hm, st.x.col_strides, st.x.col_blocks.sizes, x, h, threads=threads)
        return time.perf_counter() - t0

    probe = min(n_cells, 512)
    tp = run(probe)
    k = int(min(n_cells, max(probe, probe * 10.0 / max(tp, 1e-6))))
    t = run(k)
    frac = k / n_cells
    value = cnt["flops_hx"] * frac / t / 1e9
    return {"value": round(value, 3), "unit": "GFlop/s", "cores": threads, "kind": "port",
            "sample": f"H X on {k} of {n_cells} cells ({frac:.3f}), oracle/cellop.c "
                      f"(reference Algorithm 6, all lanes, 18 contractions), {t:.1f} s"}


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Benchmark: exact Hessian + OPG assembly of BASELINE config 1 on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Metric (BASELINE.json): Hessian/OPG entries per second.  One step assembles
the exact Hessian H and the OPG matrix G (P x P each, P = 25450) for the MLP
[784, 32, 10] (sigmoid, softmax CE) on N = 1000 seeded synthetic examples,
so a step produces 2 * P^2 matrix entries.

  value  device-resident inputs, CUDA-event timed over exactly K steps
  e2e    the same job through the host-buffer C-ABI (curvkit_assemble_*_f32):
         host->device upload of params/x/y and device->host download of H and
         G are inside the timed region
  roofline  the dominant kernel's algorithmic FLOPs / its event-timed
         duration (library-internal CUDA events on the launching stream)
  cpu_baseline  the reference library (oracle/_ref, compiled from the
         unmodified reference sources) on a bounded sample of the same job

--impl reference runs only the reference CPU arm (rank 0; other ranks exit).
Multi-GPU (torchrun), no collective on the data path either way:
  --scaling weak (default)  the units are independent curvature jobs: rank r
         assembles H and G of its own config-1 instance (parameters drawn with
         seed + r); value = N * 2 P^2 / max-over-ranks step time
  --scaling strong  one job: rank r assembles rows curvkit_shard_rows(P, N, r)
         of H and G (lower-triangle entries and their mirrors, shards balanced
         by triangle area); value = 2 P^2 / max-over-ranks step time
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PREC_DTYPE = {"tf32": "tf32", "tf32x3": "tf32x3", "f32": "f32", "f64": "f64"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c1")
    ap.add_argument("--precision", default="tf32", choices=list(PREC_DTYPE))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=4)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.lines = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx or None, "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- reference arm

def reference_sample(wl, threads, budget_s=12.0):
    """Time the reference library (oracle/_ref) on a bounded sample of the
    step: Hessian columns (its own HVP-on-basis loop, `threads` lanes) and OPG
    rows (its own rank-1 update loop); extrapolate to the full 2 P^2 job."""
    import numpy as np

    from oracle.oracle import Oracle, Ref
    params, x, y, _ = wl.draw()
    spec = dict(widths=wl.widths, activation=wl.activation)
    P = wl.P
    if Ref.available():
        lib, kind = Ref(), "reference"
    else:  # the reference tree was not built here: the C restatement
        lib, kind = Oracle(), "port"
    if kind == "port":
        raise RuntimeError("oracle/_ref missing; build it with `make -C oracle`")
    # Hessian columns spread over the parameter blocks, `threads` lanes
    ncol = threads
    c0 = 0
    t = time.perf_counter()
    lib.hessian_columns_sample(spec, params, x, y, c0, c0 + ncol, threads)
    th = time.perf_counter() - t
    t = time.perf_counter()
    lib.jacobian(spec, params, x, y)
    tj = time.perf_counter() - t
    nrow = 4 * threads
    t = time.perf_counter()
    lib.opg_rows_sample(spec, params, x, y, 0, nrow, threads)
    tr = max(1e-9, time.perf_counter() - t - tj)
    t_full = th * P / ncol + tj + tr * P / nrow
    return {
        "value": 2.0 * P * P / t_full,
        "unit": "entries/s",
        "cores": threads,
        "kind": kind,
        "sample": (f"{ncol} Hessian columns (HVP on basis vectors, {threads} lanes) + {nrow} OPG rows "
                   f"({threads} threads) of config {wl.name} (N={wl.n}, P={P}); full-job time extrapolated "
                   f"linearly: {t_full:.1f} s"),
        "seconds": th + tj + tr,
    }


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_1905_05559_b200.workloads import CONFIGS
    wl = CONFIGS[args.config]
    threads = os.cpu_count() or 1
    vals = []
    for i in range(args.warmup + args.steps):
        r = reference_sample(wl, threads)
        if i >= args.warmup:
            vals.append(r)
    v = sum(r["value"] for r in vals) / len(vals)
    ms = 2.0 * wl.P * wl.P / v * 1e3
    line = {
        "impl": "reference", "metric": "hessian_opg_entries_per_s", "value": v, "unit": "entries/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE config shapes and distributions)",
        "config": {"workload": f"{wl.name}: MLP {wl.widths} {wl.activation}, N={wl.n}, P={wl.P}, exact H + OPG",
                   "products": "hessian+opg"},
        "cpu_baseline": {"value": v, "unit": "entries/s", "cores": threads, "kind": vals[0]["kind"],
                         "sample": vals[0]["sample"]},
        "e2e": {"value": v, "unit": "entries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- B200 arm

def row_range(P, rank, world):
    per = (P + world - 1) // world
    return min(P, rank * per), min(P, (rank + 1) * per)


def run_b200(args):
    import numpy as np
    import torch

    from paper_1905_05559_b200 import _lib, curv
    from paper_1905_05559_b200.workloads import CONFIGS

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = CONFIGS[args.config]
    weak = world > 1 and args.scaling == "weak"
    if weak and rank > 0:  # an independent instance of the same config per rank
        import dataclasses
        wl = dataclasses.replace(wl, seed=wl.seed + 7919 * rank)
    prec = args.precision
    dt = torch.float64 if prec == "f64" else torch.float32
    dev = torch.device("cuda", local)
    params, x, y, labels = wl.draw()
    P, n = wl.P, wl.n
    spec = curv.ModelSpec(wl.widths, wl.activation)
    p_d = torch.tensor(params, dtype=dt, device=dev)
    x_d = torch.tensor(x, dtype=dt, device=dev)
    l_d = torch.tensor(labels, dtype=torch.int32, device=dev)
    ld = (P + 31) // 32 * 32
    H = torch.empty((P, ld), dtype=dt, device=dev)
    G = torch.empty((P, ld), dtype=dt, device=dev)
    stream = torch.cuda.current_stream()

    rb, re = curv.shard_rows(P, world, rank)

    def step():
        if world == 1 or weak:
            curv.dev_assemble_hessian(spec, p_d, x_d, l_d, n, H, ld, precision=prec, stream=stream)
            curv.dev_assemble_opg(spec, p_d, x_d, l_d, n, G, ld, precision=prec, stream=stream)
        else:  # this rank's triangle-balanced row shard of both products
            curv.dev_hessian_shard(spec, p_d, x_d, l_d, n, rb, re, H, ld, precision=prec, stream=stream)
            curv.dev_opg_shard(spec, p_d, x_d, l_d, n, rb, re, G, ld, precision=prec, stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    barrier()
    torch.cuda.synchronize()
    l0 = curv.launch_count()
    curv.profile_begin()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    prof = curv.profile_end()
    launches = (curv.launch_count() - l0) // args.steps
    barrier()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    # weak: every rank assembles a whole job; strong: the row shards cover one
    entries = 2.0 * P * P * (world if weak else 1)
    value = entries / (ms / 1e3)

    # e2e through the host-buffer C-ABI (pinned host outputs)
    e2e = None
    if not args.no_e2e and (world == 1 or weak):  # the host-buffer ABI assembles whole matrices
        lib = _lib.load()
        import ctypes as C
        hH = torch.empty((P, P), dtype=torch.float32, pin_memory=True)
        hG = torch.empty((P, P), dtype=torch.float32, pin_memory=True)
        xp = np.ascontiguousarray(x)
        yp = np.ascontiguousarray(y)
        pp = np.ascontiguousarray(params)
        cfg = curv.CurvatureConfig(batch_size_h=n, batch_size_g=n, memory_cap=1 << 40)._c()
        m = spec._c()
        dp = lambda a: a.ctypes.data_as(_lib.dptr)  # noqa: E731
        fp = lambda t: C.cast(t.data_ptr(), _lib.fptr)  # noqa: E731

        def e2e_step():
            _lib.check(lib.curvkit_assemble_hessian_f32(C.byref(m), dp(pp), dp(xp), dp(yp), n, C.byref(cfg),
                                                        curv.PRECISION[prec], fp(hH)))
            _lib.check(lib.curvkit_assemble_opg_f32(C.byref(m), dp(pp), dp(xp), dp(yp), n, C.byref(cfg),
                                                    curv.PRECISION[prec], fp(hG)))

        e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        te = (time.perf_counter() - t0) / args.e2e_steps
        if world > 1:
            t = torch.tensor([te], device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            te = float(t.item())
        h2d = 2 * 8 * (P + x.size + y.size) * world
        e2e = {"value": entries / te, "unit": "entries/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(2 * 4 * P * P * world), "ms_per_step": te * 1e3}

    if rank != 0:
        return
    pk, pk_kind = peaks()
    # dominant region: the one with the largest event-timed share of the step
    dom = max(prof, key=lambda k: prof[k]["ms"]) if prof else None
    roof = None
    if dom:
        r = prof[dom]
        per_launch_ms = r["ms"] / max(1, r["launches"])
        if r["flops"] > 0:
            peak = pk["bf16_tflops_sustained"] / 2.0 if prec in ("tf32", "tf32x3") else None
            achieved = r["flops"] / (r["ms"] / 1e3) / 1e12
            roof = {"bound": "tensor", "achieved": achieved, "unit": "TFLOP/s", "kernel": dom,
                    "peak": peak, "frac": (achieved / peak) if peak else None,
                    "peak_note": (f"TF32 dense = bf16 {pk_kind} sustained {pk['bf16_tflops_sustained']} / 2"
                                  if peak else "SIMT fp32/fp64 path: no tensor peak"),
                    "share_of_step": r["ms"] / args.steps / ms, "per_launch_ms": per_launch_ms,
                    "traffic": None}
        else:
            achieved = r["bytes"] / (r["ms"] / 1e3) / 1e9
            roof = {"bound": "hbm", "achieved": achieved, "unit": "GB/s", "kernel": dom, "peak": pk["hbm_gbs"],
                    "frac": achieved / pk["hbm_gbs"], "share_of_step": r["ms"] / args.steps / ms,
                    "per_launch_ms": per_launch_ms, "traffic": None}
        if dom in ("hess_symkr", "opg_symkr"):
            roof["note"] = ("flops = 2 N per symmetric-orbit value (the kernel's algorithmic work, DESIGN.md section 4); "
                            "at config 1 the kernel is bound by its TMA output stores (32/64-byte rows, "
                            "profiles/r01_c1_symkr_ncu_summary.txt), at configs 2/3 by the tensor pipe (~0.9 of peak)")
            # the same launches counted as the lower-triangle product a symmetry-blind kernel runs
            # (2 N per lower entry of the diagonal blocks): the rate the orbit scheme delivers
            if world == 1 or weak:  # whole diagonal blocks per rank
                ws = wl.widths
                lower = sum(pk * (pk + 1) / 2.0 for pk in (ws[k + 1] * (ws[k] + 1) for k in range(len(ws) - 1)))
                roof["reference_count_tflops"] = 2.0 * n * lower * args.steps / (r["ms"] / 1e3) / 1e12
        tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tfile):
            roof["traffic"] = json.load(open(tfile)).get(dom)
    kernels = {k: {"ms_per_step": v["ms"] / args.steps, "launches_per_step": v["launches"] // args.steps,
                   "tflops": (v["flops"] / (v["ms"] / 1e3) / 1e12) if v["flops"] else None,
                   "gbs": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["bytes"] else None}
               for k, v in prof.items()}
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:
            reference_sample(wl, os.cpu_count() or 1)  # warm-up sample (page faults, thread start), as the reference arm
            r = reference_sample(wl, os.cpu_count() or 1)
            cpu = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "unit": "entries/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {ex}"}
    line = {
        "metric": "hessian_opg_entries_per_s", "value": value, "unit": "entries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak" if (weak or world == 1) else "strong", "vs_baseline": None, "dtype": PREC_DTYPE[prec],
        "data": "synthetic (seeded, BASELINE config shapes and distributions)",
        "config": {"workload": f"{wl.name}: MLP {wl.widths} {wl.activation}, N={n}, P={P}, exact H + OPG "
                               f"({2 * P * P} entries per step)",
                   "products": "hessian+opg", "precision": prec,
                   "l2": "no flush: each step writes 2 x P^2 x 4 B = 5.2 GB >> 126 MB L2",
                   "parallelism": ("single GPU" if world == 1 else
                                   f"{world} GPUs, one independent config-1 job per GPU, no collective" if weak else
                                   f"{world} GPUs, triangle-balanced row shards of one job, no data-path collective")},
        "gpu_launches": int(launches),
        "roofline": roof, "kernels": kernels, "cpu_baseline": cpu, "e2e": e2e,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()

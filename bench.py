"""Benchmark of the SpAMM multiply path (BASELINE.json metric).

    python bench.py --gpus N --steps K --warmup W [--impl reference] [--workload cfgX] [--tau T]

One "step" is one SpAMM multiply (symbolic phase + numeric phase + C norms, the reference's timed
region `pkg/src/spamm/bench.py:135-145`) of the workload, operands already resident in HBM as
quadtrees.  N = 1 runs config 2 of BASELINE.json (exponential decay, n = 4096) at tau = 1e-8 with
the reference's default fine4 gating and reports the tau sweep beside it; N > 1 runs config 5
(n = 32768) with C sharded by row blocks and B all-gathered.  `value` is surviving GFLOP/s
(128 flop per executed 4x4x4 product, `numeric.py:28-29`, `:63-65`).  Inputs are seeded synthetic
matrices of the BASELINE.json laws (paper_1203_1692_b200/inputs.py).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HEADLINE_TAU = 1e-8
L2_FLUSH_BYTES = 256 << 20


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return {"hbm_gbs": float(p["hbm_gbs"]), "sm_max_mhz": float(p.get("sm_max_mhz", 1965.0)), "source": "measured"}
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback"}


class ClockSampler:
    """Samples nvidia-smi clocks and throttle reasons while the timed region runs."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int = 0):
        self.index, self.samples, self._stop, self._t = index, [], threading.Event(), None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                      "-i", str(self.index)], capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        mhz = sorted(int(s[0]) for s in self.samples if s and s[0].isdigit())
        mx = [int(s[1]) for s in self.samples if len(s) > 1 and s[1].isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for s in self.samples for n, v in zip(names, s[2:6]) if v.strip().lower() == "active"})
        return {"sm_mhz": mhz[len(mhz) // 2] if mhz else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def workload_operands(name: str):
    from paper_1203_1692_b200 import inputs
    a, b = inputs.make_operands(name)
    return a, b


# --------------------------------------------------------------------------- reference arm

def run_reference(args) -> None:
    """The reference's CPU implementation of the path, timed on the host cores.

    The reference is pure Python and cannot travel to the GPU box, so this arm times the CPU
    oracle port (oracle/spamm_oracle.c, OpenMP over product leaves, pinned bit for bit to the
    reference by tests/test_oracle_golden.py) on the same workload, tau and granularity."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as O
    name = args.workload or ("cfg2" if args.gpus == 1 else "cfg5")
    n_override = None
    if name == "cfg5":
        n_override = 8192      # largest size of the law whose step stays in the seconds range on a CPU
    from paper_1203_1692_b200 import inputs
    a_d, b_d = inputs.make_operands(name, n_override)
    ta = O.tree_from_dense(a_d)
    tb = ta if b_d is None else O.tree_from_dense(b_d)
    tau = args.tau
    times, counters, plan = [], None, None
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        plan = O.build_plan(ta, tb, tau)
        _, counters = O.execute_plan(plan, ta, tb, None, tau, args.granularity)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(dt)
    sec = float(np.mean(times))
    flops = 128 * counters.products4
    val = flops / sec / 1e9
    cores = O.num_threads()
    line = {
        "impl": "reference", "metric": "spamm_surviving_gflops", "value": val, "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": "strong" if args.gpus > 1 else "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": name, "n": int(a_d.shape[0]), "tau": tau, "granularity": args.granularity,
                   "tasks": len(plan), "products4": counters.products4},
        "cpu_baseline": {"value": val, "unit": "GFLOP/s", "cores": cores, "kind": "port",
                         "sample": f"whole {name} multiply (n={a_d.shape[0]}), C oracle with OpenMP"},
        "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# --------------------------------------------------------------------------- own arm

def timed_multiply(P, torch, qa, qb, cfg, steps, warmup, flush):
    """Per-step CUDA-event times of multiply(); L2 is flushed between steps, outside the events."""
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    out = None
    for it in range(warmup + steps):
        flush.fill_(it)
        if it >= warmup:
            ev[it - warmup][0].record()
        out = P.multiply(qa, qb, cfg)
        if it >= warmup:
            ev[it - warmup][1].record()
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev], out


def kernel_time_execute(P, torch, plan, qa, qb, cfg, reps, flush):
    """Average duration of the leaf-multiply kernel alone (CUDA events around the launch)."""
    import ctypes as C
    from paper_1203_1692_b200 import _lib
    lib = _lib.lib()
    dev = qa.device
    nC = plan.n_cleaves
    va, vb = qa.view(plan.depth), qb.view(plan.depth)
    vals = torch.empty((nC, _lib.REC), dtype=torch.float32, device=dev)
    vals_t = torch.empty_like(vals)
    leaf_sq = torch.empty((nC,), dtype=torch.float64, device=dev)
    cnt = torch.zeros((2,), dtype=torch.int64, device=dev)
    bufs = plan.buffers()
    st = torch.cuda.current_stream().cuda_stream
    times = []
    for it in range(reps + 2):
        flush.fill_(it)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(lib.spamm_execute(C.byref(va), C.byref(vb), C.byref(bufs), plan.n_steps, nC, float(cfg.tau), 1.0,
                                     0 if cfg.granularity == "fine4" else 1, 0, vals.data_ptr(), vals_t.data_ptr(),
                                     leaf_sq.data_ptr(), cnt.data_ptr(), st), "execute")
        e1.record()
        torch.cuda.synchronize()
        if it >= 2:
            times.append(e0.elapsed_time(e1))
    return float(np.mean(times))


def run_own(args) -> None:
    import torch
    import torch.distributed as dist

    import paper_1203_1692_b200 as P
    from paper_1203_1692_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    name = args.workload or ("cfg2" if world == 1 else "cfg5")
    pk = peaks()
    fp32_peak_tflops = 2 * 128 * 148 * pk["sm_max_mhz"] * 1e6 / 1e12
    a_d, b_d = workload_operands(name)
    n = a_d.shape[0]
    flush = torch.empty((L2_FLUSH_BYTES,), dtype=torch.uint8, device="cuda")
    cfg = P.MultiplyConfig(tau=args.tau, granularity=args.granularity)

    if world > 1:
        from paper_1203_1692_b200 import parallel
        result = parallel.bench_sharded(P, torch, dist, a_d, b_d, cfg, args.steps, args.warmup, flush)
        if rank == 0:
            result["line"].update({"n_gpus": world, "steps": args.steps, "warmup": args.warmup})
            print(json.dumps(result["line"]))
        dist.destroy_process_group()
        return

    qa = P.QuadtreeMatrix.from_dense(a_d)
    qb = qa if b_d is None else P.QuadtreeMatrix.from_dense(b_d)
    torch.cuda.synchronize()

    # ---- headline: K steps of multiply(), operands resident
    l0 = _lib.launch_count()
    with ClockSampler(local) as clocks:
        times, (c, plan, counters) = timed_multiply(P, torch, qa, qb, cfg, args.steps, args.warmup, flush)
    launches = (_lib.launch_count() - l0) * args.steps // (args.steps + args.warmup)
    ms = float(np.mean(times))
    p4 = counters.products4
    flops = 128 * p4 if cfg.granularity == "fine4" else 8192 * len(plan)
    value = flops / (ms * 1e-3) / 1e9

    # ---- the dominant kernel alone, for the roofline
    k3_ms = kernel_time_execute(P, torch, plan, qa, qb, cfg, max(5, args.steps), flush)
    k3_tflops = flops / (k3_ms * 1e-3) / 1e12
    # compulsory traffic of the kernel: every stored A leaf (transposed copy) and B leaf once, C leaves
    # written in both layouts, task records
    alg_bytes = 1088 * (qa.nleaf + qb.nleaf + 2 * plan.n_cleaves) + 64 * plan.n_steps

    # ---- end to end through the public API with host buffers
    host_a = torch.from_numpy(a_d).pin_memory()
    host_b = host_a if b_d is None else torch.from_numpy(b_d).pin_memory()
    host_c = torch.empty((a_d.shape[0], (b_d if b_d is not None else a_d).shape[1]), dtype=torch.float32).pin_memory()
    e2e_times = []
    for it in range(2 + max(3, args.steps // 2)):
        flush.fill_(it)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ta = P.QuadtreeMatrix.from_dense(host_a)
        tb = ta if b_d is None else P.QuadtreeMatrix.from_dense(host_b)
        cc, _, _ = P.multiply(ta, tb, cfg)
        host_c.copy_(cc.to_dense_tensor(), non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        if it >= 2:
            e2e_times.append(e0.elapsed_time(e1))
    e2e_ms = float(np.mean(e2e_times))
    h2d = a_d.nbytes * (1 if b_d is None else 2)

    # ---- tau sweep (config 2 of BASELINE.json), both granularities
    sweep = []
    if not args.no_sweep:
        from paper_1203_1692_b200 import inputs
        taus = inputs.WORKLOADS[name].taus
        ref64 = None
        if n <= 8192:
            ad = torch.from_numpy(a_d).cuda().double()
            bd = ad if b_d is None else torch.from_numpy(b_d).cuda().double()
            ref64 = ad @ bd
            del ad, bd
        for tau in taus:
            for gran in ("fine4", "coarse16"):
                cf = P.MultiplyConfig(tau=tau, granularity=gran)
                ts, (cs, pl, ks) = timed_multiply(P, torch, qa, qb, cf, 5, 2, flush)
                fl = 128 * ks.products4 if gran == "fine4" else 8192 * len(pl)
                kt = kernel_time_execute(P, torch, pl, qa, qb, cf, 5, flush)
                err = None
                if ref64 is not None:
                    err = float((cs.to_dense_tensor().double() - ref64).abs().max().item())
                L = 1 << pl.depth
                sweep.append({"tau": tau, "granularity": gran, "ms": float(np.median(ts)), "tasks": len(pl),
                              "task_fraction": len(pl) / float(L) ** 3, "products4": ks.products4,
                              "gflops": fl / (np.median(ts) * 1e-3) / 1e9, "kernel_ms": kt,
                              "kernel_tflops": fl / (kt * 1e-3) / 1e12,
                              "kernel_frac_fp32_peak": fl / (kt * 1e-3) / 1e12 / fp32_peak_tflops,
                              "max_abs_err_vs_fp64": err})
        del ref64

    # ---- CPU baseline beside it: the oracle port on the host cores
    cpu = None
    if not args.no_cpu:
        from oracle import oracle as O
        ta_o = O.tree_from_dense(a_d)
        tb_o = ta_o if b_d is None else O.tree_from_dense(b_d)
        t0 = time.perf_counter()
        opl = O.build_plan(ta_o, tb_o, args.tau)
        _, ocnt = O.execute_plan(opl, ta_o, tb_o, None, args.tau, args.granularity)
        dt = time.perf_counter() - t0
        cpu = {"value": 128 * ocnt.products4 / dt / 1e9, "unit": "GFLOP/s", "cores": O.num_threads(), "kind": "port",
               "sample": f"one whole {name} multiply, {dt:.2f} s (C oracle port of the reference, OpenMP)"}

    line = {
        "metric": "spamm_surviving_gflops", "value": value, "unit": "GFLOP/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": name, "n": int(n), "tau": args.tau, "granularity": args.granularity,
                   "tasks": len(plan), "product_leaves": plan.n_cleaves, "products4": p4,
                   "l2": f"flushed between steps ({L2_FLUSH_BYTES >> 20} MiB write)",
                   "effective_gflops_2n3": 2.0 * n ** 3 / (ms * 1e-3) / 1e9},
        "roofline": {"bound": "fp32", "kernel": "execute_kernel", "achieved": k3_tflops, "peak": fp32_peak_tflops,
                     "unit": "TFLOP/s", "frac": k3_tflops / fp32_peak_tflops,
                     "peak_source": f"2*128 lanes*148 SMs*{pk['sm_max_mhz']:.0f} MHz ({pk['source']} clock)",
                     "kernel_ms": k3_ms, "traffic": None,
                     "hbm_frac_of_measured": alg_bytes / (k3_ms * 1e-3) / 1e9 / pk["hbm_gbs"]},
        "cpu_baseline": cpu,
        "e2e": {"value": flops / (e2e_ms * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(host_c.numel() * 4)},
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
        "sweep": sweep,
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="own", choices=("own", "reference"))
    ap.add_argument("--workload", default=None)
    ap.add_argument("--tau", type=float, default=HEADLINE_TAU)
    ap.add_argument("--granularity", default="fine4", choices=("fine4", "coarse16"))
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_own(args)


if __name__ == "__main__":
    main()

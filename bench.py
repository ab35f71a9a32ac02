"""Benchmark of the SpAMM multiply path (BASELINE.json metric).

    python bench.py --gpus N --steps K --warmup W [--impl reference] [--workload cfgX] [--tau T]

One "step" is one SpAMM multiply (symbolic phase + numeric phase + C norms, the reference's timed
region `pkg/src/spamm/bench.py:135-145`) of the workload, operands already resident in HBM as
quadtrees.  N = 1 runs config 2 of BASELINE.json (exponential decay, n = 4096) at tau = 1e-8 with
the reference's default fine4 gating and reports the tau sweep and the other configs beside it;
N > 1 (under torchrun) runs config 5 (n = 32768) with C sharded by row blocks and the operand
shards all-gathered inside the timed region.  `value` is surviving GFLOP/s (128 flop per executed
4x4x4 product, `numeric.py:28-29`, `:63-65`).  Inputs are seeded synthetic matrices of the
BASELINE.json laws (paper_1203_1692_b200/inputs.py).
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
NUM_SMS = 148      # B200; replaced by the device's count once a GPU is visible (run_single)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return {"hbm_gbs": float(p["hbm_gbs"]), "sm_max_mhz": float(p.get("sm_max_mhz", 1965.0)), "source": "measured"}
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback"}


def recorded_traffic(workload: str, granularity: str):
    """dram bytes per launch of execute_kernel from the committed `ncu --set full` capture."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(f"{workload}:{granularity}")
    except (OSError, ValueError):
        return None


class ClockSampler:
    """Samples SM clocks and throttle reasons while the timed region runs (NVML, every 2 ms;
    `nvidia-smi --query-gpu` as the fallback)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int = 0):
        self.index, self.mhz, self.max_mhz, self.reasons = index, [], None, set()
        self._stop, self._t, self._nvml, self._h = threading.Event(), None, None, None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self._physical_index(index))
            self.max_mhz = int(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self._nvml = None

    @staticmethod
    def _physical_index(index: int) -> int:
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            ids = [v.strip() for v in vis.split(",") if v.strip()]
            if index < len(ids) and ids[index].isdigit():
                return int(ids[index])
        return index

    def _sample_nvml(self):
        n = self._nvml
        self.mhz.append(int(n.nvmlDeviceGetClockInfo(self._h, n.NVML_CLOCK_SM)))
        r = int(n.nvmlDeviceGetCurrentClocksEventReasons(self._h)) if hasattr(n, "nvmlDeviceGetCurrentClocksEventReasons") \
            else int(n.nvmlDeviceGetCurrentClocksThrottleReasons(self._h))
        for name, bit in (("hw_slowdown", 0x8), ("sw_power_cap", 0x4), ("sw_thermal_slowdown", 0x20),
                          ("hw_thermal_slowdown", 0x40)):
            if r & bit:
                self.reasons.add(name)

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-i",
                              str(self.index)], capture_output=True, text=True, timeout=5).stdout.strip()
        s = [x.strip() for x in out.split(",")]
        if len(s) >= 6 and s[0].isdigit():
            self.mhz.append(int(s[0]))
            if s[1].isdigit():
                self.max_mhz = max(self.max_mhz or 0, int(s[1]))
            for name, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), s[2:6]):
                if v.lower() == "active":
                    self.reasons.add(name)

    def _run(self):
        while not self._stop.is_set():
            try:
                if self._nvml is not None:
                    self._sample_nvml()
                else:
                    self._sample_smi()
            except Exception:
                pass
            self._stop.wait(0.002 if self._nvml is not None else 0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        mhz = sorted(self.mhz)
        return {"sm_mhz": mhz[len(mhz) // 2] if mhz else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(mhz),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


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
    from paper_1203_1692_b200 import inputs
    name = args.workload or ("cfg2" if args.gpus == 1 else "cfg5")
    n_override = None
    sample = f"whole {name} multiply"
    if name == "cfg5":
        n_override = 8192      # largest size of the law whose step stays in the seconds range on a CPU
        sample = "cfg5 law at n=8192 (n=32768 does not fit the time bound on a CPU)"
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
    flops = 128 * counters.products4 if args.granularity == "fine4" else 8192 * len(plan)
    val = flops / sec / 1e9
    cores = O.num_threads()
    line = {
        "impl": "reference", "metric": "spamm_surviving_gflops", "value": val, "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": "strong" if args.gpus > 1 else "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": name, "n": int(a_d.shape[0]), "tau": tau, "granularity": args.granularity,
                   "tasks": len(plan), "product_leaves": int(np.unique(plan.c_keys).size), "products4": counters.products4,
                   "l2": "not applicable (CPU arm)",
                   "effective_gflops_2n3": 2.0 * float(a_d.shape[0]) ** 3 / sec / 1e9},
        "cpu_baseline": {"value": val, "unit": "GFLOP/s", "cores": cores, "kind": "port",
                         "sample": f"{sample}; C port of the reference algorithm, OpenMP over product leaves",
                         "python_reference": python_reference_time(name, tau, args.granularity)},
        "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# --------------------------------------------------------------------------- own arm, one GPU

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
    va, vb = qa.view(plan.depth), qb.view(plan.depth, left=False)
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


def kernel_time_plan(P, torch, plan, qa, qb, tau, reps, flush):
    """Average duration of the symbolic phase alone (spamm_plan: plan_tiles + plan_order kernels,
    plus root/expand for deep trees), CUDA events around the C call, L2 flushed."""
    import ctypes as C
    from paper_1203_1692_b200 import _lib
    from paper_1203_1692_b200.symbolic import PlanAlloc
    lib = _lib.lib()
    va, vb = qa.view(plan.depth), qb.view(plan.depth, left=False)
    pb = PlanAlloc(qa.device, plan.depth, max(plan.n_steps, 1) + 64, max(plan.n_cleaves, 1) + 64)
    st = torch.cuda.current_stream().cuda_stream
    times = []
    for it in range(reps + 2):
        flush.fill_(it)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(lib.spamm_plan(C.byref(va), C.byref(vb), float(tau), 0, 1 << plan.depth, C.byref(pb.struct),
                                  pb.ws.data_ptr(), pb.ws_bytes, st), "plan")
        e1.record()
        torch.cuda.synchronize()
        if it >= 2:
            times.append(e0.elapsed_time(e1))
    assert int(pb.counts[2].item()) == 0 and int(pb.counts[4].item()) == plan.n_steps
    return float(np.mean(times))


def kernel_time_interior(P, torch, c, reps, flush):
    """Average duration of the interior-norm kernel on the product tree (K4, compute_norms on C)."""
    from paper_1203_1692_b200 import _lib
    lib = _lib.lib()
    depth = c.depth
    cells, total = 1 << (2 * depth), _lib.level_total(depth)
    dev = c.device
    g = c.grids()
    sq_grid = torch.zeros((cells,), dtype=torch.float64, device=dev)
    off = _lib.level_offset(depth)
    leaf_norm = g.norm[off:off + cells].double()
    sq_grid.copy_(torch.where(leaf_norm >= 0, leaf_norm * leaf_norm, torch.zeros_like(leaf_norm)))
    norm, norm_t = g.norm.clone(), g.norm_t.clone()
    sq_levels = torch.empty((total,), dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    times = []
    for it in range(reps + 2):
        flush.fill_(it)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(lib.spamm_build_interior(sq_grid.data_ptr(), depth, norm.data_ptr(), norm_t.data_ptr(),
                                            sq_levels.data_ptr(), 0, st), "build_interior")
        e1.record()
        torch.cuda.synchronize()
        if it >= 2:
            times.append(e0.elapsed_time(e1))
    return float(np.mean(times))


def time_from_dense(P, torch, dense_dev, reps, flush):
    """Average duration of QuadtreeMatrix.from_dense on a device-resident dense matrix (K1: leaf and
    sub-block norms, slot scan, leaf packing in both layouts, interior norms)."""
    times, q = [], None
    for it in range(reps + 2):
        flush.fill_(it)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        q = P.QuadtreeMatrix.from_dense(dense_dev)
        e1.record()
        torch.cuda.synchronize()
        if it >= 2:
            times.append(e0.elapsed_time(e1))
        if it < reps + 1:
            del q
    return float(np.mean(times)), q


def python_reference_time(name: str, tau: float, gran: str):
    """Seconds per multiply of the unmodified Python reference, measured in the build container by
    profiles/python_reference_time.py (the reference cannot run on the GPU box)."""
    try:
        with open(os.path.join(ROOT, "profiles", "python_reference_times.json")) as f:
            d = json.load(f)
        r = d["runs"].get(f"{name}:{tau:g}:{gran}")
        if r:
            return {"multiply_s": r["multiply_s"], "build_plan_s": r["build_plan_s"], "execute_plan_s": r["execute_plan_s"],
                    "from_dense_s": r["from_dense_s"], "cores": 1, "where": d["where"], "when": d["when"]}
    except (OSError, ValueError, KeyError):
        pass
    return None


def touched_leaves(torch, plan, nleaf_a: int, nleaf_b: int):
    """Distinct stored leaves of A and of B that occur in at least one task of the plan (SURVEY.md 8d:
    the operand part of the numeric kernel's compulsory traffic), counted on the device from the
    step records."""
    st = plan.steps[: plan.n_steps].to(torch.int64) & 0xFFFFFFFF

    def popc16(x):
        x = x - ((x >> 1) & 0x5555)
        x = (x & 0x3333) + ((x >> 2) & 0x3333)
        x = (x + (x >> 4)) & 0x0F0F
        return (x + (x >> 8)) & 0x1F

    def pos(r, c):          # Morton position of leaf (r, c) inside its 4x4 block
        return ((r >> 1) << 3) | ((c >> 1) << 2) | ((r & 1) << 1) | (c & 1)

    rowmask = [sum(1 << pos(d, c) for c in range(4)) for d in range(4)]
    colmask = [sum(1 << pos(r, d) for r in range(4)) for d in range(4)]
    hit_a = torch.zeros((max(nleaf_a, 1),), dtype=torch.bool, device=st.device)
    hit_b = torch.zeros((max(nleaf_b, 1),), dtype=torch.bool, device=st.device)
    a_first, a_present, b_first, b_present = st[:, 4], st[:, 5], st[:, 6], st[:, 7]
    for kk in range(4):
        live = st[:, 8 + kk]
        for d in range(4):
            use = (live & rowmask[d]) != 0
            hit_a[(a_first + popc16(a_present & ((1 << pos(d, kk)) - 1)))[use]] = True
            use = (live & colmask[d]) != 0
            hit_b[(b_first + popc16(b_present & ((1 << pos(kk, d)) - 1)))[use]] = True
    return int(hit_a.sum().item()), int(hit_b.sum().item())


def measure_case(P, torch, qa, qb, tau, gran, flush, fp32_peak, ref64=None, steps=5, hbm_gbs=None):
    cf = P.MultiplyConfig(tau=tau, granularity=gran)
    ts, (cs, pl, ks) = timed_multiply(P, torch, qa, qb, cf, steps, 3, flush)
    fl = 128 * ks.products4 if gran == "fine4" else 8192 * len(pl)
    kt = kernel_time_execute(P, torch, pl, qa, qb, cf, steps, flush)
    err = None
    if ref64 is not None:
        err = float((cs.to_dense_tensor().double() - ref64).abs().max().item())
    L = 1 << pl.depth
    med = float(np.median(ts))
    # compulsory traffic of the leaf-multiply kernel: every operand leaf that occurs in a task once, the
    # product leaves in both layouts, the step records
    ta_hit, tb_hit = touched_leaves(torch, pl, qa.nleaf, qb.nleaf)
    alg_bytes = 1088 * (ta_hit + tb_hit + 2 * pl.n_cleaves) + 64 * pl.n_steps
    out = {"tau": tau, "granularity": gran, "ms": med, "tasks": len(pl), "task_fraction": len(pl) / float(L) ** 3,
           "products4": ks.products4, "product_leaves": pl.n_cleaves, "gflops": fl / (med * 1e-3) / 1e9, "kernel_ms": kt,
           "kernel_tflops": fl / (kt * 1e-3) / 1e12, "kernel_frac_fp32_peak": fl / (kt * 1e-3) / 1e12 / fp32_peak,
           "kernel_algorithmic_bytes": int(alg_bytes), "operand_leaves_in_tasks": [ta_hit, tb_hit],
           "max_abs_err_vs_fp64": err}
    if hbm_gbs:
        out["kernel_frac_hbm_peak"] = alg_bytes / (kt * 1e-3) / 1e9 / hbm_gbs
    return out


def run_single(args, torch, P, local: int) -> None:
    from paper_1203_1692_b200 import _lib, inputs
    global NUM_SMS
    name = args.workload or "cfg2"
    pk = peaks()
    NUM_SMS = torch.cuda.get_device_properties(local).multi_processor_count
    fp32_peak = 2 * 128 * NUM_SMS * pk["sm_max_mhz"] * 1e6 / 1e12
    a_d, b_d = inputs.make_operands(name)
    n = a_d.shape[0]
    flush = torch.empty((L2_FLUSH_BYTES,), dtype=torch.uint8, device="cuda")
    cfg = P.MultiplyConfig(tau=args.tau, granularity=args.granularity)
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
    k3_ms = kernel_time_execute(P, torch, plan, qa, qb, cfg, max(5, min(args.steps, 50)), flush)
    k3_tflops = flops / (k3_ms * 1e-3) / 1e12
    # compulsory traffic of the kernel: every A leaf (transposed copy) and B leaf that occurs in a task
    # once, C leaves written in both layouts, step records
    ta_hit, tb_hit = touched_leaves(torch, plan, qa.nleaf, qb.nleaf)
    alg_bytes = 1088 * (ta_hit + tb_hit + 2 * plan.n_cleaves) + 64 * plan.n_steps
    n_tasks, n_cleaves = len(plan), plan.n_cleaves

    # ---- the other kernels of the path, each against the roofline that bounds it
    reps_k = max(5, min(args.steps, 20))
    k2_ms = kernel_time_plan(P, torch, plan, qa, qb, cfg.tau, reps_k, flush)
    k4_ms = kernel_time_interior(P, torch, c, reps_k, flush)
    dense_dev = torch.from_numpy(a_d).cuda()
    k1_ms, _q = time_from_dense(P, torch, dense_dev, reps_k, flush)
    del _q, dense_dev
    n_p = 16 << qa.depth
    La = 1 << qa.depth
    # K1: the dense matrix read once, the stored leaves written in both record layouts, the grids and pyramid
    k1_bytes = 4 * n * n + 2 * 1088 * qa.nleaf + La * La * (4 + 4 + 4 + 4 + 8) * 4 // 3
    # K2: the leaf norm grids of both operands (and their sub-norm range grids) read once, one record per step written
    k2_bytes = (4 + 4) * (La * La) * 2 + 64 * plan.n_steps + 4 * 4 * plan.counts[5].item()
    # K4: C's leaf grid of square sums read, every level of both norm pyramids and the square sums written
    Lc = 1 << c.depth
    k4_bytes = Lc * Lc * 8 + Lc * Lc * (4 + 4 + 8) * 4 // 3

    # ---- end to end through the public API with host buffers
    # The operands are host trees in the reference's packed form (keys + 16x16 leaf blocks, the arrays
    # of packed_leaves(), `core.py:387-405`: what the reference arm's timed region starts from as well);
    # the result comes back as the product tree's packed leaves (keys + 272-float leaf records), not as
    # a zero-filled dense matrix.  The variant that starts from a dense host matrix is reported beside it.
    cap = plan.n_cleaves
    host_vals = torch.empty((cap, _lib.REC), dtype=torch.float32).pin_memory()
    host_keys = torch.empty((cap,), dtype=torch.int32).pin_memory()

    def packed_host(q):
        k, v, _s = q.packed_leaves()
        return torch.from_numpy(k.astype(np.int32)).pin_memory(), torch.from_numpy(v.reshape(-1, 256)).pin_memory()

    pk_a = packed_host(qa)
    pk_b = pk_a if b_d is None else packed_host(qb)
    host_a = torch.from_numpy(a_d).pin_memory()
    host_b = host_a if b_d is None else torch.from_numpy(b_d).pin_memory()

    def e2e_time(step):
        times, d2h_bytes = [], 0
        for it in range(2 + max(3, min(args.steps, 20) // 2)):
            flush.fill_(it)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            cc = step()
            nc = cc.nleaf                       # reads the counts back (the one synchronisation of the step)
            host_vals[:nc].copy_(cc.values[:nc], non_blocking=True)
            host_keys[:nc].copy_(cc.keys[:nc], non_blocking=True)
            d2h_bytes = nc * (_lib.REC * 4 + 4)
            e1.record()
            torch.cuda.synchronize()
            if it >= 2:
                times.append(e0.elapsed_time(e1))
        return float(np.mean(times)), d2h_bytes

    def step_packed():
        ta = P.QuadtreeMatrix.from_packed(n, n, pk_a[0], pk_a[1])
        tb = ta if b_d is None else P.QuadtreeMatrix.from_packed(n, n, pk_b[0], pk_b[1])
        return P.multiply(ta, tb, cfg)[0]

    def step_dense():
        ta = P.QuadtreeMatrix.from_dense(host_a)
        tb = ta if b_d is None else P.QuadtreeMatrix.from_dense(host_b)
        return P.multiply(ta, tb, cfg)[0]

    # operands that stay on the host (paper_1203_1692_b200.hosttree): keys, norms and sub-block norms go up, the
    # plan is made, and the GPU fetches only the leaves that occur in a surviving task from pinned host memory
    h_a = P.HostTree.from_device(qa)
    h_b = None if b_d is None else P.HostTree.from_device(qb)
    fetched_box = {}

    def step_host():
        cc, _, _, fetched = P.multiply_host(h_a, h_b, cfg)
        fetched_box["n"] = fetched
        return cc

    # the same in two blocks of rows of C: block 1 is copied back (side stream) while block 2 is planned, fetched and
    # multiplied, so that PCIe runs in both directions at once; no synchronisation before the end of the step
    side = torch.cuda.Stream()
    part_bufs = {}

    def e2e_time_parts(nparts):
        times, d2h_bytes = [], 0
        for it in range(2 + max(3, min(args.steps, 20) // 2)):
            flush.fill_(it)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sizes = []

            def copy_back(part):
                (r0, r1), cc, _plan, _k, _f = part
                vals, keys = cc.values, cc.keys          # capacity-bounded views: the leaf count is still on the device
                hv = part_bufs.get((r0, "v"))
                if hv is None or hv.shape[0] < vals.shape[0]:
                    hv = part_bufs[(r0, "v")] = torch.empty(tuple(vals.shape), dtype=vals.dtype).pin_memory()
                    part_bufs[(r0, "k")] = torch.empty((vals.shape[0],), dtype=torch.int32).pin_memory()
                ev = torch.cuda.Event()
                ev.record()
                side.wait_event(ev)
                with torch.cuda.stream(side):
                    hv[: vals.shape[0]].copy_(vals, non_blocking=True)
                    part_bufs[(r0, "k")][: keys.shape[0]].copy_(keys, non_blocking=True)
                sizes.append(int(vals.shape[0]) * (_lib.REC * 4 + 4))

            res = P.multiply_host_parts(h_a, h_b, cfg, parts=nparts, on_part=copy_back)
            torch.cuda.current_stream().wait_stream(side)
            e1.record()
            torch.cuda.synchronize()
            fetched_box["parts"] = sum(int(p[4].sum().item()) for p in res)
            d2h_bytes = sum(sizes)
            if it >= 2:
                times.append(e0.elapsed_time(e1))
        return float(np.mean(times)), d2h_bytes

    e2e_dense_ms, _ = e2e_time(step_dense)
    e2e_packed_ms, _ = e2e_time(step_packed)
    e2e_one_ms, d2h_one = e2e_time(step_host)
    e2e_two_ms, d2h_two = e2e_time_parts(2)
    if e2e_one_ms <= e2e_two_ms:      # the better schedule is the headline; both are reported
        e2e_ms, d2h, e2e_parts = e2e_one_ms, d2h_one, 1
    else:
        e2e_ms, d2h, e2e_parts = e2e_two_ms, d2h_two, 2
    fetched_leaves = int(fetched_box["n"].sum().item()) if e2e_parts == 1 else int(fetched_box["parts"])
    h2d_host = h_a.skeleton_bytes() + (0 if h_b is None else h_b.skeleton_bytes()) + fetched_leaves * 1024
    h2d = sum(int(t.numel()) * t.element_size() for t in pk_a) * (1 if b_d is None else 2)
    h2d_dense = a_d.nbytes * (1 if b_d is None else 2)

    # ---- tau sweep of the headline workload (config 2 of BASELINE.json), both granularities
    sweep = []
    if not args.no_sweep:
        ref64 = None
        if n <= 8192:
            ad = torch.from_numpy(a_d).cuda().double()
            bd = ad if b_d is None else torch.from_numpy(b_d).cuda().double()
            ref64 = ad @ bd
            del ad, bd
        for tau in inputs.WORKLOADS[name].taus:
            for gran in ("fine4", "coarse16"):
                sweep.append(measure_case(P, torch, qa, qb, tau, gran, flush, fp32_peak, ref64, hbm_gbs=pk["hbm_gbs"]))
        del ref64

    # ---- CPU baseline beside it: the oracle port on the host cores
    cpu = None
    if not args.no_cpu:
        from oracle import oracle as O
        ta_o = O.tree_from_dense(a_d)
        tb_o = ta_o if b_d is None else O.tree_from_dense(b_d)
        reps, t0 = 0, time.perf_counter()
        while reps < 3 or (time.perf_counter() - t0 < 10.0 and reps < 200):
            opl = O.build_plan(ta_o, tb_o, args.tau)
            _, ocnt = O.execute_plan(opl, ta_o, tb_o, None, args.tau, args.granularity)
            reps += 1
        dt = (time.perf_counter() - t0) / reps
        oflops = 128 * ocnt.products4 if args.granularity == "fine4" else 8192 * len(opl)
        cpu = {"value": oflops / dt / 1e9, "unit": "GFLOP/s", "cores": O.num_threads(), "kind": "port",
               "sample": f"{reps} whole {name} multiplies, {dt * 1e3:.1f} ms each (C port of the reference "
                         f"algorithm, OpenMP over product leaves)",
               "python_reference": python_reference_time(name, args.tau, args.granularity)}
        del ta_o, tb_o

    # ---- the other BASELINE.json configs on this GPU (time per multiply, GFLOP/s, K3 fraction)
    others = []
    if not args.no_configs and args.workload is None:
        del qa, qb, c, plan
        for wl in ("cfg1", "cfg3", "cfg4", "cfg5"):
            xa, xb = inputs.make_operands(wl)
            ta = P.QuadtreeMatrix.from_dense(xa)
            tb = ta if xb is None else P.QuadtreeMatrix.from_dense(xb)
            nn = int(xa.shape[0])
            del xa, xb
            for tau in inputs.WORKLOADS[wl].taus:
                for gran in ("fine4", "coarse16"):
                    r = measure_case(P, torch, ta, tb, tau, gran, flush, fp32_peak, None, steps=3, hbm_gbs=pk["hbm_gbs"])
                    r.update({"workload": wl, "n": nn})
                    others.append(r)
            del ta, tb
            torch.cuda.empty_cache()

    # ---- time and rate against n (the metric's other axis): the config-2 law at tau = 1e-8
    n_sweep = []
    if not args.no_configs and args.workload is None:
        for nn in (1024, 2048, 8192, 16384):
            xa, _ = inputs.make_operands("cfg2", nn)
            ta = P.QuadtreeMatrix.from_dense(xa)
            del xa
            for gran in ("fine4", "coarse16"):
                r = measure_case(P, torch, ta, ta, HEADLINE_TAU, gran, flush, fp32_peak, None, steps=3, hbm_gbs=pk["hbm_gbs"])
                r.update({"workload": "cfg2 law", "n": nn, "effective_gflops_2n3": 2.0 * nn ** 3 / (r["ms"] * 1e-3) / 1e9})
                n_sweep.append(r)
            del ta
            torch.cuda.empty_cache()

    line = {
        "metric": "spamm_surviving_gflops", "value": value, "unit": "GFLOP/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": name, "n": int(n), "tau": args.tau, "granularity": args.granularity,
                   "tasks": n_tasks, "product_leaves": n_cleaves, "products4": p4,
                   "l2": f"flushed between steps ({L2_FLUSH_BYTES >> 20} MiB write)",
                   "effective_gflops_2n3": 2.0 * n ** 3 / (ms * 1e-3) / 1e9},
        "roofline": {"bound": "fp32", "kernel": "execute_kernel", "achieved": k3_tflops, "peak": fp32_peak,
                     "unit": "TFLOP/s", "frac": k3_tflops / fp32_peak,
                     "peak_source": f"2*128 lanes*{NUM_SMS} SMs*{pk['sm_max_mhz']:.0f} MHz ({pk['source']} max clock); "
                                    "MEASURED_PEAKS.json has no FP32 FMA figure",
                     "kernel_ms": k3_ms, "traffic": recorded_traffic(name, args.granularity),
                     "algorithmic_bytes": int(alg_bytes),
                     "hbm_frac_of_measured": alg_bytes / (k3_ms * 1e-3) / 1e9 / pk["hbm_gbs"]},
        "roofline_k1": {"bound": "hbm", "kernel": "from_dense (leaf_norms_dense + slot scan + pack_leaves + interior)",
                        "achieved": k1_bytes / (k1_ms * 1e-3) / 1e9, "peak": pk["hbm_gbs"], "unit": "GB/s",
                        "frac": k1_bytes / (k1_ms * 1e-3) / 1e9 / pk["hbm_gbs"], "ms": k1_ms, "algorithmic_bytes": int(k1_bytes)},
        "roofline_k2": {"bound": "latency (hbm shown)", "kernel": "spamm_plan (plan_tiles + plan_order)",
                        "achieved": k2_bytes / (k2_ms * 1e-3) / 1e9, "peak": pk["hbm_gbs"], "unit": "GB/s",
                        "frac": k2_bytes / (k2_ms * 1e-3) / 1e9 / pk["hbm_gbs"], "ms": k2_ms, "algorithmic_bytes": int(k2_bytes)},
        "roofline_k4": {"bound": "latency (hbm shown)", "kernel": "interior_kernel (norms of C)",
                        "achieved": k4_bytes / (k4_ms * 1e-3) / 1e9, "peak": pk["hbm_gbs"], "unit": "GB/s",
                        "frac": k4_bytes / (k4_ms * 1e-3) / 1e9 / pk["hbm_gbs"], "ms": k4_ms, "algorithmic_bytes": int(k4_bytes)},
        "cpu_baseline": cpu,
        "e2e": {"value": flops / (e2e_ms * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": int(h2d_host), "d2h_bytes_per_step": int(d2h),
                "operands": "host trees (HostTree: the arrays of packed_leaves() + leaf norms, pinned); multiply_host sends keys and "
                            "norms, plans, and the GPU fetches the leaves that occur in a task from host memory",
                "operand_leaves_fetched": fetched_leaves,
                "row_blocks": e2e_parts,
                "one_block": {"ms_per_step": e2e_one_ms, "d2h_bytes_per_step": int(d2h_one)},
                "two_row_blocks": {"ms_per_step": e2e_two_ms, "d2h_bytes_per_step": int(d2h_two),
                                   "note": "block 1 copied back on a side stream while block 2 is fetched and multiplied"},
                "result": "product tree as packed leaves (keys + leaf records)",
                "all_leaves": {"value": flops / (e2e_packed_ms * 1e-3) / 1e9, "ms_per_step": e2e_packed_ms,
                               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                               "operands": "every stored leaf uploaded first (keys + 16x16 blocks, pinned), QuadtreeMatrix.from_packed"},
                "from_dense": {"value": flops / (e2e_dense_ms * 1e-3) / 1e9, "ms_per_step": e2e_dense_ms,
                               "h2d_bytes_per_step": int(h2d_dense), "d2h_bytes_per_step": int(d2h),
                               "operands": "dense host matrix (pinned), QuadtreeMatrix.from_dense"}},
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
        "sweep": sweep,
        "configs": others,
        "n_sweep": n_sweep,
    }
    print(json.dumps(line))


# --------------------------------------------------------------------------- own arm, N GPUs

def run_sharded(args, torch, dist, P, local: int) -> None:
    """Config 5 with C's leaf rows split across the ranks.  The rank's rows of A are resident as a
    tree (as the operands are at N = 1).  Timed region of one step, per rank: exchange of the packed
    leaves (B = A) -> tree of B (grids and pyramid only) -> fused multiply, which yields the own rows
    of C.  The row blocks are cut by surviving-task count once, at set-up.  The end-to-end figure
    starts from the host rows instead and builds everything."""
    from paper_1203_1692_b200 import _lib, inputs, parallel
    rank, world = dist.get_rank(), dist.get_world_size()
    name = args.workload or "cfg5"
    cfg = P.MultiplyConfig(tau=args.tau, granularity=args.granularity)
    flush = torch.empty((L2_FLUSH_BYTES,), dtype=torch.uint8, device="cuda")

    # rank 0 draws the matrix and builds the tree; the packed leaves are broadcast (set-up, untimed)
    meta = torch.zeros((4,), dtype=torch.int64, device="cuda")
    if rank == 0:
        a_d, b_d = inputs.make_operands(name)
        if b_d is not None:
            raise SystemExit("the sharded bench runs C = A*A workloads (cfg2, cfg4, cfg5)")
        q0 = P.QuadtreeMatrix.from_dense(a_d)
        meta[:] = torch.tensor([a_d.shape[0], a_d.shape[1], q0.nleaf, 0])
        del a_d
    dist.broadcast(meta, 0)
    m, n, nleaf = int(meta[0]), int(meta[1]), int(meta[2])
    if rank == 0:
        whole = parallel.shard_of_tree(q0, 0, 1 << 30)
        del q0
    else:
        whole = parallel.PackedShard(torch.empty((nleaf,), dtype=torch.int32, device="cuda"),
                                     torch.empty((nleaf, 272), dtype=torch.float32, device="cuda"),
                                     torch.empty((nleaf,), dtype=torch.float64, device="cuda"))
    for t in (whole.keys, whole.records, whole.leaf_sq):
        dist.broadcast(t, 0)
    full = parallel.tree_from_shard(m, n, whole)
    nrows = -(-m // 16)
    # the partition of A's rows is the partition of the work: cut by surviving-task count (set-up, untimed)
    from paper_1203_1692_b200.symbolic import build_plan
    probe = build_plan(full, full, cfg.tau)
    counts = parallel.row_task_counts(probe, probe.depth).cpu().numpy()
    splits = parallel.balanced_row_split(counts[:nrows], world)
    r0, r1 = splits[rank]
    del probe
    mine = parallel.shard_of_tree(full, r0, r1)
    host_rows = full.to_dense_tensor()[r0 * 16:min(m, r1 * 16)].cpu().pin_memory()
    del full, whole
    torch.cuda.empty_cache()

    mine_tree = parallel.tree_from_shard(m, n, mine)       # the resident form of the local rows, as at N = 1

    # the headline step: everything about the exchange that needs the host is prepared once (ShardedMultiply);
    # the step is exchange (asynchronous) + interior rows meanwhile + the remaining rows afterwards
    chosen = "auto" if args.exchange == "auto" else args.exchange
    sm = parallel.ShardedMultiply(mine, None, (m, n), (m, n), cfg, splits=splits, exchange=chosen, overlap=True,
                                  a_tree=mine_tree)

    def step_resident():
        return sm.run()

    host_out = {}

    def step_e2e():
        shard = parallel.shard_from_dense_rows(host_rows, r0)
        c, plan, counters = parallel.multiply_sharded(shard, None, (m, n), (m, n), cfg, exchange=sm.exchange,
                                                      splits=splits)
        nc = c.nleaf                         # this rank's product leaves, read back as packed leaves
        if host_out.get("vals") is None or host_out["vals"].shape[0] < nc:
            host_out["vals"] = torch.empty((nc, 272), dtype=torch.float32).pin_memory()
            host_out["keys"] = torch.empty((nc,), dtype=torch.int32).pin_memory()
        host_out["vals"][:nc].copy_(c.values[:nc], non_blocking=True)
        host_out["keys"][:nc].copy_(c.keys[:nc], non_blocking=True)
        host_out["bytes"] = nc * (272 * 4 + 4)
        return c, plan, counters

    def timed(fn, steps, warmup):
        times, out = [], None
        for it in range(warmup + steps):
            flush.fill_(it)
            dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = fn()
            e1.record()
            torch.cuda.synchronize()
            if it >= warmup:
                times.append(e0.elapsed_time(e1))
        t = torch.tensor([float(np.mean(times))], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()), out

    l0 = _lib.launch_count()
    with ClockSampler(local) as clocks:
        ms, parts = timed(step_resident, args.steps, args.warmup)
    launches = (_lib.launch_count() - l0) * args.steps // (args.steps + args.warmup)
    work = torch.tensor([float(sum(k.products4 for _, _, _, k in parts)), float(sum(len(p) for _, _, p, _ in parts)),
                         float(r1 - r0), float(sum(c.nleaf for _, c, _, _ in parts))], dtype=torch.float64, device="cuda")

    # the alternatives beside it, each prepared the same way (N > 1 only: with one rank they coincide)
    variants = {}
    if world > 1:
        for label, ex, ov in (("allgather", "all", False), ("allgather_overlap", "all", True),
                              ("needed", "needed", False), ("needed_overlap", "needed", True)):
            alt = parallel.ShardedMultiply(mine, None, (m, n), (m, n), cfg, splits=splits, exchange=ex, overlap=ov,
                                           a_tree=mine_tree)
            t_alt, _ = timed(alt.run, max(2, min(args.steps, 10)), 3)
            variants[label] = {"ms_per_step": t_alt}
            del alt
    per_rank = [torch.zeros_like(work) for _ in range(world)]
    dist.all_gather(per_rank, work)
    tot_p4 = sum(float(w[0]) for w in per_rank)
    tot_tasks = sum(float(w[1]) for w in per_rank)
    flops = 128.0 * tot_p4 if cfg.granularity == "fine4" else 8192.0 * tot_tasks
    e2e_ms, _ = timed(step_e2e, max(2, min(args.steps, 5)), 2)
    # for reference: the same step with B already replicated (no exchange, trees prebuilt)
    from paper_1203_1692_b200.numeric import multiply_async
    a_local = mine_tree
    b_have = parallel.tree_from_shard(m, n, parallel.allgather_shards(mine), transposed=False)
    local_ms, _ = timed(lambda: multiply_async(a_local, b_have, cfg, None), max(2, min(args.steps, 10)), 3)
    # the dominant kernel on this rank's rows, alone (as at N = 1): rank 0's figure goes into the line
    c_r, plan_r, k_r = multiply_async(a_local, b_have, cfg, None, row_range=(r0, r1))
    torch.cuda.synchronize()
    k3_ms = kernel_time_execute(P, torch, plan_r, a_local, b_have, cfg, max(3, min(args.steps, 10)), flush)
    k3_flops = 128.0 * k_r.products4 if cfg.granularity == "fine4" else 8192.0 * len(plan_r)
    pk = peaks()
    fp32_peak = 2 * 128 * torch.cuda.get_device_properties(local).multi_processor_count * pk["sm_max_mhz"] * 1e6 / 1e12
    d2h = host_out.get("bytes", 0)
    io = torch.tensor([float(host_rows.numel() * 4), float(d2h)], dtype=torch.float64, device="cuda")
    dist.all_reduce(io)
    if rank == 0:
        line = {
            "metric": "spamm_surviving_gflops", "value": flops / (ms * 1e-3) / 1e9, "unit": "GFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": name, "n": m, "tau": args.tau, "granularity": args.granularity,
                       "tasks": int(tot_tasks), "products4": int(tot_p4),
                       "parallelism": f"row blocks of A and C x{world} cut by task count; exchange of B inside the timed "
                                      f"region: {'all-gather' if sm.exchange == 'all' else 'needed leaf rows only'} (NCCL, "
                                      f"{'chosen automatically, ' if args.exchange == 'auto' else ''}rank 0 needs "
                                      f"{sm.need_fraction:.2f} of B's leaf rows), interior rows {sm.interior} of {sm.rows} "
                                      "multiplied while the exchange is in flight",
                       "with_exchange": {"ms_per_step": ms, "exchange": sm.exchange, "overlap": True},
                       "exchange_variants": variants,
                       "without_exchange": {"ms_per_step": local_ms, "value": flops / (local_ms * 1e-3) / 1e9,
                                            "note": "B already replicated, trees prebuilt: the local multiply alone"},
                       "tasks_per_rank": [int(w[1]) for w in per_rank],
                       "l2": f"flushed between steps ({L2_FLUSH_BYTES >> 20} MiB write)"},
            "roofline": {"bound": "fp32", "kernel": "execute_kernel on rank 0's rows, timed alone", "achieved": k3_flops / (k3_ms * 1e-3) / 1e12,
                         "peak": fp32_peak, "unit": "TFLOP/s", "frac": k3_flops / (k3_ms * 1e-3) / 1e12 / fp32_peak,
                         "peak_source": f"2*128 lanes*SMs*{pk['sm_max_mhz']:.0f} MHz ({pk['source']} max clock); MEASURED_PEAKS.json has no FP32 FMA figure",
                         "kernel_ms": k3_ms, "traffic": None},
            "cpu_baseline": None,        # rank 0 at N = 1 only (bench contract)
            "e2e": {"value": flops / (e2e_ms * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": int(io[0].item()), "d2h_bytes_per_step": int(io[1].item())},
            "gpu_launches": int(launches), "clocks": clocks.summary(),
        }
        return line
    return None


def run_own(args) -> None:
    import torch
    import torch.distributed as dist

    if not os.path.exists(os.path.join(ROOT, "paper_1203_1692_b200", "csrc", "libspamm_b200.so")):
        if int(os.environ.get("LOCAL_RANK", "0")) == 0:     # a bare checkout: compile the library once
            import __graft_entry__
            __graft_entry__.build()

    import paper_1203_1692_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    sharded = world > 1 or os.environ.get("SPAMM_BENCH_SHARDED") == "1"
    if sharded:
        if not dist.is_initialized():
            if "MASTER_ADDR" not in os.environ:
                os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": "29531", "RANK": "0", "WORLD_SIZE": "1"})
            # NCCL writes its log (at least the version banner) to stdout; the JSON line must be the only one there
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        # ... and whatever else a library prints while the ranks run: file descriptor 1 points at stderr until the
        # line itself is written
        sys.stdout.flush()
        real_stdout = os.dup(1)
        os.dup2(2, 1)
        line = None
        try:
            if not dist.is_initialized():
                dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            line = run_sharded(args, torch, dist, P, local)
        finally:
            if dist.is_initialized():
                dist.destroy_process_group()
            sys.stdout.flush()
            os.dup2(real_stdout, 1)
            os.close(real_stdout)
        if line is not None:
            print(json.dumps(line))
    else:
        run_single(args, torch, P, local)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="own", choices=("own", "reference"))
    ap.add_argument("--workload", default=None)
    ap.add_argument("--tau", type=float, default=HEADLINE_TAU)
    ap.add_argument("--granularity", default="fine4", choices=("fine4", "coarse16"))
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--exchange", default=os.environ.get("SPAMM_EXCHANGE", "auto"), choices=("auto", "all", "needed"),
                    help="N > 1: bring all of B to every rank (all-gather), only the leaf rows it reaches, or decide "
                         "by the share of B the rank needs (auto: needed when below half)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_own(args)


if __name__ == "__main__":
    main()

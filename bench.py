"""Benchmark: MVC time-to-solution on the 1M-vertex planted-cover graph
(BASELINE.json configs[3], the config the metric's 1/2/4/8-GPU scaling is
quoted on), with the other configs as secondary measurements.

One step = one ``solve(g, SolverConfig())`` MVC call through the package's
public API on the planted1m instance: the grid-wide root fixpoint, crown,
device compaction and (when anything is left) the persistent search kernel.
``value`` is the time-to-solution with the input CSR already resident in
HBM; ``e2e`` repeats the step from pinned host buffers (upload, solve,
result readback inside the timed region).  ``other_configs`` holds
configs[0]-[2] (er200 MVC, the rgg2000 PVC pair with its search-tree
nodes/s, ba100k MVC).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

N > 1 runs under torchrun, one rank per GPU; rank r solves its own seeded
instance of the same shape (seed 1 + r: independent objects, weak scaling),
and ``value`` is the max over ranks.  ``--impl reference`` times the
reference algorithm's CPU implementation (the C restatement in oracle/, its
threaded engine on every host core) on the same workload; that arm never
imports the product package (the generators are loaded from synth.py by
path), so no CUDA library is mapped into it.
"""

from __future__ import annotations

import argparse
import importlib.util
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MVC time-to-solution (s) & search-tree nodes/s at 1/2/4/8 B200 vs CPU ref"
WORKLOAD = ("configs[3]: MVC on a 1M-vertex sparse synthetic graph (planted cover of 50,000 "
            "plus noise)")
GENERATOR = ("synth.planted(n=1_000_000, cover=50_000, cc=1.0, oo=0.3, seed=1+rank): every "
             "outside vertex attaches to 2-3 random cover vertices, 50,000 random cover-cover "
             "edges, 300,000 random outside-outside noise edges; the reference's root rules "
             "resolve it completely (no search-tree nodes), so its time-to-solution is the "
             "root pipeline's")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true")
    ap.add_argument("--no-strong", action="store_true")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def load_synth():
    """synth.py by path: plain numpy generators, no package import."""
    spec = importlib.util.spec_from_file_location(
        "vc_synth", os.path.join(ROOT, "paper_2512_18334_b200", "synth.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def instance(seed):
    return load_synth().planted(1_000_000, 50_000, seed)


def config(world, n, m):
    """Identical in both arms (same N)."""
    return {"workload": WORKLOAD, "generator": GENERATOR, "n": n, "m": m,
            "parallelism": (f"{world} GPUs, independent seeded instances (weak scaling)"
                            if world > 1 else "1 GPU"),
            "l2": "inputs (31 MB CSR) well below L2 size: L2 flushed between timed steps "
                  "(512 MiB write outside the timed region)"}


# --------------------------------------------------------------- clocks ----

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def _nvml_loop(self, nv, h):
        """NVML every 2 ms (nvidia-smi -lms prints every ~100 ms, so a 15 ms
        timed region often held no sample); same line format."""
        R = (nv.nvmlClocksThrottleReasonHwSlowdown, nv.nvmlClocksThrottleReasonHwThermalSlowdown,
             nv.nvmlClocksThrottleReasonSwThermalSlowdown, nv.nvmlClocksThrottleReasonSwPowerCap)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self.stop:
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                util = nv.nvmlDeviceGetUtilizationRates(h).gpu
            except nv.NVMLError:
                break
            self.lines.append(", ".join([str(sm), str(mx)] +
                                        ["Active" if rs & r else "Not Active" for r in R] +
                                        [str(util)]))
            time.sleep(0.002)

    def __enter__(self):
        self.stop = False
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.source = "nvml (2 ms)"
            self.t = threading.Thread(target=self._nvml_loop, args=(nv, h), daemon=True)
            self.t.start()
            deadline = time.time() + 3.0
            while len(self.lines) < 2 and time.time() < deadline:
                time.sleep(0.005)
            if self.lines:
                return self
        except Exception:  # no NVML: nvidia-smi below
            self.stop = True
        self.source = "nvidia-smi -lms 20"
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi takes a while to print its first sample: the timed
            # region starts only once it is streaming
            deadline = time.time() + 3.0
            while len(self.lines) < 2 and time.time() < deadline:
                time.sleep(0.01)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self.stop = True
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def mark_start(self):
        self.w0 = len(self.lines)

    def mark_end(self):
        # the first sample after the window closes is the nearest one when
        # the timed region is shorter than nvidia-smi's sampling period
        self.w1 = len(self.lines)
        deadline = time.time() + 1.0
        while len(self.lines) <= self.w1 and time.time() < deadline and self.proc:
            time.sleep(0.01)

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        w0, w1 = getattr(self, "w0", 0), getattr(self, "w1", len(self.lines))
        window = self.lines[w0:max(w1, w0 + 1)]
        for ln in window:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
            except ValueError:
                continue
            for nm, val in zip(names, p[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm),
                "samples_in_window": max(0, w1 - w0), "source": getattr(self, "source", None)}


# ------------------------------------------------------------ reference ----

def run_reference(args):
    """The reference algorithm's CPU implementation (oracle/, threaded engine
    on every host core) on the same workload; rank 0 only."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle

    n, off, nbr = instance(1)
    cores = os.cpu_count() or 1
    opt = None

    def step():
        nonlocal opt
        t = time.perf_counter()
        r = oracle.solve(n, off, nbr, workers=cores)
        dt = time.perf_counter() - t
        if opt is None:
            opt = r["cover_size"]
        elif r["cover_size"] != opt:
            raise RuntimeError("reference arm: unstable answer")
        return dt, r["stats"]["tree_nodes_visited"]

    for _ in range(args.warmup):
        step()
    total, nodes = 0.0, 0
    for _ in range(args.steps):
        dt, nd = step()
        total += dt
        nodes += nd
    tts = total / args.steps
    line = {
        "impl": "reference", "metric": METRIC, "value": tts, "unit": "s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tts * 1e3, "time_to_solution_s": tts, "nodes_per_s": nodes / total,
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic (seeded planted-cover graph, seed 1)",
        "config": config(world, n, int(off[-1]) // 2),
        "answer": {"mvc": opt},
        "cpu_baseline": {"value": tts, "unit": "s", "cores": cores, "kind": "port",
                         "sample": f"{args.steps} MVC solves of planted1m seed 1 "
                                   f"(oracle/vc_oracle.c, threaded engine, {cores} threads; "
                                   f"the root pipeline is sequential)"},
        "e2e": {"value": tts, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ b200 ----

def cpu_baseline_sample():
    """oracle/ (single-thread C port of the reference) on a bounded sample."""
    import oracle

    n, off, nbr = instance(1)
    reps, t0 = 0, time.perf_counter()
    while reps < 5 and (reps == 0 or time.perf_counter() - t0 < 10.0):
        oracle.solve(n, off, nbr, deterministic=True)
        reps += 1
    dt = time.perf_counter() - t0
    return {"value": dt / reps, "unit": "s", "cores": 1, "kind": "port",
            "sample": f"{reps} MVC solves of planted1m seed 1, single-thread C restatement "
                      f"(oracle/vc_oracle.c), {dt:.1f} s"}


def load_capture():
    """The committed ncu --set full capture of the root kernel (one planted1m
    launch): dram bytes per launch, L2 traffic and atomic rates."""
    p = os.path.join(ROOT, "profiles", "r02_root_front_ncu.json")
    try:
        with open(p) as f:
            return json.load(f), os.path.relpath(p, ROOT)
    except (OSError, ValueError):
        return {}, None


def atomic_frac(cap):
    """L2 atomic requests/s of the captured launch against the measured L2
    atomic peak (profiles/r02_l2_atomic_peak.json: distinct-address ATOM,
    tools/l2_atomic_peak.cu on this pool's B200)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_l2_atomic_peak.json")) as f:
            peak = json.load(f)["ATOM distinct"]["G_atomics_per_s"] * 1e9
    except (OSError, ValueError, KeyError):
        return None
    rate = cap.get("l2_atomic_requests_per_s") if cap else None
    return {"achieved_per_s": rate, "peak_per_s": peak,
            "frac": rate / peak if rate else None,
            "peak_source": "profiles/r02_l2_atomic_peak.json (ATOM, distinct addresses)"}


def other_configs(vc, torch, reps=5):
    """configs[0]-[2] through the public API, device-timed with CUDA events."""
    synth = load_synth()
    out = {}

    def timed(fn):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1), r

    for key, name, gen in (
            ("configs[0]", "er200 MVC: G(n=200, avg degree 4), seed 1", lambda: synth.er(200, 4.0, 1)),
            ("configs[2]", "ba100k MVC: synth.ba(100_000, m=3, seed 1) -- Barabasi-Albert with 2 % "
                           "single-edge arrivals (pure m=3 BA has minimum degree 3 and nothing for "
                           "the root rules to start from)", lambda: synth.ba(100_000, 3, 1)),
            ("configs[3] variant", "planted1m MVC with 3x the noise (synth.planted(oo=1.0)): the "
                                   "root rules leave a residual to search",
             lambda: synth.planted(1_000_000, 50_000, 1, oo=1.0))):
        n, off, nbr = gen()
        g = vc.StaticGraph(n, off, nbr)
        vc.solve(g)
        ms = []
        for _ in range(reps):
            t, r = timed(lambda: vc.solve(g))
            ms.append(t)
        out[key] = {"workload": name, "mvc": r.cover_size,
                    "time_to_solution_s": statistics.median(ms) * 1e-3,
                    "tree_nodes": r.stats.tree_nodes_visited}
    n, off, nbr = synth.rgg(2000, 0.027, 1)
    g = vc.StaticGraph(n, off, nbr)
    opt = vc.solve(g).cover_size
    cfgs = [vc.SolverConfig(mode="pvc", k=opt), vc.SolverConfig(mode="pvc", k=opt - 1)]
    vc.solve_batch(g, cfgs)
    pair_ms, pair_nodes, single = [], 0, {opt: [], opt - 1: []}
    for _ in range(reps * 4):
        t, rs = timed(lambda: vc.solve_batch(g, cfgs))
        assert rs[0].found and not rs[1].found
        pair_ms.append(t)
        pair_nodes += sum(r.stats.tree_nodes_visited for r in rs)
    for k in single:
        for _ in range(reps * 2):
            t, r = timed(lambda: vc.solve(g, vc.SolverConfig(mode="pvc", k=k)))
            single[k].append((t, r.stats.tree_nodes_visited))
    for key, name, gen in (("configs[4] gnp400", "MVC G(n=400, p=0.1), 2 s budget",
                            lambda: synth.gnp(400, 0.1, 1)),
                           ("configs[4] torus60", "MVC torus 60x60, 2 s budget",
                            lambda: synth.torus(60, 60)),
                           ("configs[2] pure BA", "MVC pure Barabasi-Albert n=100k m=3 "
                            "(synth.ba(pendant=0)), 2 s budget",
                            lambda: synth.ba(100_000, 3, 1, pendant=0.0))):
        n4, off4, nbr4 = gen()
        g4 = vc.StaticGraph(n4, off4, nbr4)
        vc.solve(g4, vc.SolverConfig(timeout=0.2))
        t, r = timed(lambda: vc.solve(g4, vc.SolverConfig(timeout=2.0)))
        out[key] = {"workload": name + " (beyond exact search on either side: nodes/s and the "
                                      "best cover reached)",
                    "best_cover": r.cover_size, "exact": r.exact,
                    "tree_nodes": r.stats.tree_nodes_visited,
                    "nodes_per_s": r.stats.tree_nodes_visited / (t * 1e-3),
                    "warp_tier_share": r.warp_nodes / max(1, r.stats.tree_nodes_visited)}
    out["configs[1]"] = {
        "workload": "PVC yes/no pair (k=opt, opt-1) on random geometric graph n=2000 r=0.027",
        "opt": opt,
        "pair_solve_batch_s": statistics.median(pair_ms) * 1e-3,
        "pair_nodes_per_s": pair_nodes / (sum(pair_ms) * 1e-3),
        "single_query_time_to_solution_s": {
            f"k={k}": statistics.median(t for t, _ in v) * 1e-3 for k, v in single.items()},
        "single_query_nodes_per_s": {
            f"k={k}": sum(nd for _, nd in v) / (sum(t for t, _ in v) * 1e-3)
            for k, v in single.items()},
    }
    return out


STRONG = {"n": 180, "p": 0.08, "seed": 1, "mvc": 136, "subtrees": 128}


def strong_scaling(vc, torch, world, ndev, barrier, steps=2):
    """ONE hard instance across all ranks (distributed.solve_distributed:
    subtrees from the store's ticket counter, in-flight bound exchange):
    time-to-solution and search-tree nodes/s at this N.  The instance is the
    configs[4] family (dense-ish Erdos-Renyi) at the size whose exact MVC one
    GPU proves in seconds; its optimum is pinned by the C oracle
    (tests/golden/strong.json)."""
    from paper_2512_18334_b200.distributed import solve_distributed

    synth = load_synth()
    per = -(-STRONG["subtrees"] // world)  # the same total partition at every N
    n, off, nbr = synth.gnp(STRONG["n"], STRONG["p"], STRONG["seed"])
    g = vc.StaticGraph(n, off, nbr)

    def one():
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = solve_distributed(g, vc.SolverConfig(), subtrees_per_rank=per)
        e1.record()
        torch.cuda.synchronize()
        if r.cover_size != STRONG["mvc"] or not r.exact:
            raise RuntimeError(f"strong instance: MVC {r.cover_size}, expected {STRONG['mvc']}")
        return e0.elapsed_time(e1), r.stats.tree_nodes_visited

    one()  # warm-up
    ms, nodes = 0.0, 0
    for _ in range(steps):
        t, nd = one()
        ms += t
        nodes += nd
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda" if world <= ndev else "cpu")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms = float(tt[0])
    tts = ms / steps * 1e-3
    return {"workload": f"MVC on G(n={STRONG['n']}, p={STRONG['p']}), seed {STRONG['seed']} "
                        f"(configs[4] family, exact): one instance across all {world} GPU(s)",
            "n_gpus": world, "scaling": "strong", "steps": steps, "warmup": 1,
            "time_to_solution_s": tts, "nodes_per_s": nodes / (ms * 1e-3),
            "tree_nodes_per_solve": nodes / steps, "mvc": STRONG["mvc"],
            "subtrees": STRONG["subtrees"], "subtrees_per_rank": per,
            "timing": "CUDA events around solve_distributed, max over ranks"}


def run_b200(args):
    import numpy as np
    import torch

    rank, world, local = dist_env()
    ndev = torch.cuda.device_count()
    device = local % ndev
    torch.cuda.set_device(device)
    import paper_2512_18334_b200 as vc
    from paper_2512_18334_b200 import _lib

    _lib.set_device(device)
    if world > 1:
        import torch.distributed as dist

        if world <= ndev:
            dist.init_process_group("nccl", device_id=torch.device("cuda", device))
        else:  # fewer GPUs than ranks: a functional run of the multi-process path
            dist.init_process_group("gloo")
    n, off, nbr = instance(1 + rank)
    m = int(off[-1]) // 2
    g = vc.StaticGraph(n, off, nbr)
    opt = vc.solve(g, vc.SolverConfig()).cover_size  # untimed: the answer every step must give
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    # pinned host copies of the input for the end-to-end leg
    off_pin = torch.empty(len(off), dtype=torch.int64, pin_memory=True).numpy()
    nbr_pin = torch.empty(len(nbr), dtype=torch.int32, pin_memory=True).numpy()
    off_pin[:] = off
    nbr_pin[:] = nbr

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def step(graph):
        r = vc.solve(graph, vc.SolverConfig())
        if r.cover_size != opt or not r.exact:
            raise RuntimeError(f"MVC {r.cover_size}, expected {opt}")
        return r

    clk = ClockSampler(device).__enter__()  # running before the timed region
    for _ in range(args.warmup):
        step(g)
    barrier()
    l0 = _lib.launch_count()
    total_ms, nodes = 0.0, 0
    kern_ms, kern_launches, kern_scans, kind = 0.0, 0, 0, None
    kern_sweeps, kern_bars, kern_walked = 0, 0, 0
    clk.mark_start()
    for _ in range(args.steps):
        flush.zero_()  # L2 flush between timed steps (outside the events)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = step(g)
        e1.record()
        torch.cuda.synchronize()
        total_ms += e0.elapsed_time(e1)
        nodes += r.stats.tree_nodes_visited
        kern_ms += r.root_kernel.get("ms", 0.0)
        kern_launches += r.root_kernel.get("launches", 0)
        kern_scans += r.root_kernel.get("scans", 0)
        kern_sweeps += r.root_kernel.get("sweeps", 0)
        kern_bars += r.root_kernel.get("barriers", 0)
        kern_walked += r.root_kernel.get("walked", 0)
        kind = r.root_kernel.get("kind")
    clk.mark_end()
    launches = _lib.launch_count() - l0

    # e2e: from pinned host buffers every step (upload + solve + readback)
    e2e_ms = 0.0
    for _ in range(args.steps):
        flush.zero_()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gh = vc.StaticGraph(n, off_pin, nbr_pin)
        r = step(gh)
        e1.record()
        torch.cuda.synchronize()
        e2e_ms += e0.elapsed_time(e1)
        del gh
    clk.__exit__(None, None, None)
    h2d = off_pin.nbytes + nbr_pin.nbytes
    rn, rm = r.stats.root_vertices_after, 0
    pre_forced = len(r.forced_ids)
    # per solve the host reads back the vertex map, the reduced CSR (int32)
    # and the result structs; the forced ids stay on the device with the
    # reduced graph until first use (SolveResult.forced_ids is lazy)
    d2h = 8 * rn + 4 * (rn + 1) + 8 * rm + 512

    strong = None if args.no_strong else strong_scaling(vc, torch, world, ndev, barrier)

    t = torch.tensor([total_ms, e2e_ms, nodes], dtype=torch.float64,
                     device="cuda" if world <= ndev else "cpu")
    if world > 1:
        tmax = t.clone()
        torch.distributed.all_reduce(tmax, op=torch.distributed.ReduceOp.MAX)
        tsum = t.clone()
        torch.distributed.all_reduce(tsum, op=torch.distributed.ReduceOp.SUM)
        total_ms, e2e_ms, nodes = float(tmax[0]), float(tmax[1]), float(tsum[2])
    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return

    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except (OSError, ValueError):
        pass
    peak = peaks.get("hbm_gbs") or 7672.0
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if peaks.get("hbm_gbs") else \
        "fallback (B200_PROFILING.md)"
    # algorithmic bytes of one root-fixpoint launch ("Kernels"):
    # what any fixpoint must touch -- the CSR read once (int32 offsets +
    # neighbours) and the int32 degree array written and read once
    L = max(kern_launches, 1)
    per_launch_scans = kern_scans / L
    alg_bytes = 4 * (n + 1) + 8 * m + 8 * n
    launch_ms = kern_ms / L
    achieved = alg_bytes / (launch_ms * 1e-3) / 1e9 if launch_ms else 0.0
    cap, traffic_src = load_capture()
    traffic = cap.get("dram_bytes_per_launch")
    tts = total_ms / args.steps * 1e-3
    line = {
        "metric": METRIC,
        "value": tts,
        "unit": "s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps,
        "time_to_solution_s": tts,
        "nodes_per_s": nodes / (total_ms * 1e-3),
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "int32",
        "data": "synthetic (seeded planted-cover graph, seed 1 + rank)",
        "config": config(world, n, m),
        "answer": {"mvc": opt, "tree_nodes_per_solve": nodes / args.steps / world,
                   "root_forced": pre_forced, "reduced_vertices": rn},
        "e2e": {"value": e2e_ms / args.steps * 1e-3, "unit": "s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_ms / args.steps,
                "input": "pinned host numpy arrays (int64 offsets, int32 neighbours)"},
        "gpu_launches": launches,
        "roofline": {
            "bound": "hbm", "kernel": f"k_root_front (root fixpoint, kind={kind})",
            "achieved": achieved, "peak": peak, "peak_source": peak_src, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
            "algorithmic_bytes_per_launch": alg_bytes, "full_passes_per_launch": per_launch_scans,
            "launch_ms": launch_ms, "launches_per_step": kern_launches / args.steps,
            "kernel_share_of_step": kern_ms / total_ms if total_ms else None,
            # what binds it: sequential sweeps (the reference's sweep order)
            # separated by grid barriers, each a few L2 round trips deep
            "l2_atomic_frac": atomic_frac(cap),
            "l2_from_capture": {k: cap.get(k) for k in (
                "l2_bytes", "l2_gbs", "l2_sector_throughput_pct_of_peak", "l2_atomic_requests",
                "l2_atomic_requests_per_s", "l2_atomic_unit_active_pct_of_peak",
                "issue_active_pct", "top_stalls_per_issue")} if cap else None,
            "latency": {"sweeps_per_launch": kern_sweeps / L,
                        "grid_barriers_per_launch": kern_bars / L,
                        "adjacency_entries_walked_per_launch": kern_walked / L,
                        "us_per_barrier_interval": (launch_ms * 1e3 / (kern_bars / L)
                                                    if kern_bars else None)},
        },
        "clocks": clk.summary(),
    }
    if strong is not None:
        line["strong_scaling"] = strong
    if not args.no_other_configs:
        line["other_configs"] = other_configs(vc, torch)
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_sample()
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()

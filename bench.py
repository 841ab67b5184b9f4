"""Benchmark: PVC yes/no pair on the 2,000-vertex random geometric graph
(BASELINE.json configs[1]) -- time-to-solution and search-tree nodes/s.

One step = the batch {PVC k=opt, PVC k=opt-1} through the package's public
API (solve_batch: the two independent queries run concurrently, each with
its own host thread, stream and half of the resident block slots; root
reduction, compaction and the persistent search kernel all on the device).  `value` is whole-job search-tree nodes/s with the input CSR
already resident in HBM; `e2e` repeats the step from host numpy buffers
(upload, solve, result readback inside the timed region).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

N > 1 runs under torchrun, one rank per GPU; rank r solves its own seeded
instance of the same shape (seed 1 + r: independent objects, weak scaling).
--impl reference times the reference algorithm's CPU implementation (the C
restatement in oracle/, threaded, every host core) on the same workload.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MVC time-to-solution (s) & search-tree nodes/s at 1/2/4/8 B200 vs CPU ref"
WORKLOAD = "PVC yes/no pair (k=opt, k=opt-1) on random geometric graph n=2000 r=0.027"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mode", default="weak", choices=["weak", "strong"],
                    help="weak: each rank solves its own seeded instance; strong: all ranks "
                         "solve instance 1 together (root-subtree partition + bound exchange)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def instance(seed):
    from paper_2512_18334_b200 import synth

    return synth.rgg(2000, 0.027, seed)


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

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
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
                "samples_in_window": max(0, w1 - w0)}


# ------------------------------------------------------------ reference ----

def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle

    n, off, nbr = instance(1)
    cores = os.cpu_count() or 1
    opt = oracle.solve(n, off, nbr, deterministic=True)["cover_size"]

    def step():
        nodes = 0
        for k, want in ((opt, True), (opt - 1, False)):
            r = oracle.solve(n, off, nbr, mode="pvc", k=k, workers=cores)
            assert r["found"] == want, (k, r["found"])
            nodes += r["stats"]["tree_nodes_visited"]
        return nodes

    for _ in range(args.warmup):
        step()
    nodes, t0 = 0, time.perf_counter()
    for _ in range(args.steps):
        nodes += step()
    dt = time.perf_counter() - t0
    value = nodes / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "nodes/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic (seeded RGG)",
        "config": {"workload": WORKLOAD, "seed": 1, "opt": opt},
        "cpu_baseline": {"value": value, "unit": "nodes/s", "cores": cores, "kind": "port",
                         "sample": f"{args.steps} PVC pairs on rgg2000 seed 1 "
                                   f"(oracle/vc_oracle.c threaded engine, {cores} threads)"},
        "e2e": {"value": value, "unit": "nodes/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ b200 ----

def cpu_baseline_sample():
    """oracle/ (single-thread C port of the reference) on a bounded sample."""
    import oracle

    n, off, nbr = instance(1)
    opt = oracle.solve(n, off, nbr, deterministic=True)["cover_size"]
    nodes, reps, t0 = 0, 0, time.perf_counter()
    while reps < 5 and (reps == 0 or time.perf_counter() - t0 < 10.0):
        for k in (opt, opt - 1):
            nodes += oracle.solve(n, off, nbr, mode="pvc", k=k, deterministic=True)[
                "stats"]["tree_nodes_visited"]
        reps += 1
    dt = time.perf_counter() - t0
    return {"value": nodes / dt, "unit": "nodes/s", "cores": 1, "kind": "port",
            "sample": f"{reps} PVC pairs (k=opt, opt-1) on rgg2000 seed 1, single-thread "
                      f"C restatement (oracle/vc_oracle.c), {dt:.1f} s",
            "ms_per_pair": dt / reps * 1e3}


def load_traffic():
    """dram bytes per search-kernel launch from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "search_kernel_ncu.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), d
    except (OSError, ValueError):
        return None, None


def run_b200(args):
    import numpy as np
    import torch

    rank, world, local = dist_env()
    # one rank per GPU; ranks only share a GPU when there are fewer GPUs than
    # ranks (a functional test of the multi-process path), then over gloo
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
        else:
            dist.init_process_group("gloo")
    strong = args.mode == "strong" and world > 1
    n, off, nbr = instance(1 if strong else 1 + rank)
    g = vc.StaticGraph(n, off, nbr)
    opt = vc.solve(g, vc.SolverConfig()).cover_size  # untimed: defines the pair
    if strong:
        from paper_2512_18334_b200.distributed import solve_distributed
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def pair(graph):
        # the step's two PVC queries are independent: solve_batch runs them
        # concurrently (own host thread, stream and half the block slots each)
        nodes = kms = 0.0
        ks = ((opt, True), (opt - 1, False))
        if strong:
            rs = [solve_distributed(graph, vc.SolverConfig(mode="pvc", k=k)) for k, _ in ks]
        else:
            rs = vc.solve_batch(graph, [vc.SolverConfig(mode="pvc", k=k) for k, _ in ks])
        for (k, want), r in zip(ks, rs):
            if r.found != want:
                raise RuntimeError(f"PVC k={k}: found={r.found}, expected {want}")
            nodes += r.stats.tree_nodes_visited
            kms += r.search_ms
        return nodes, kms

    # per-solve record traffic comes from the search result; wrap solve once
    from paper_2512_18334_b200 import engine as _eng

    rec = {"bytes": 0, "kernel_ms": 0.0, "launches": 0}
    orig = _eng.run_search

    rec_lock = threading.Lock()  # solve_batch calls it from worker threads

    def run_search_probe(*a, **kw):
        out = orig(*a, **kw)
        res = out[0]
        with rec_lock:
            rec["bytes"] += (res.records_loaded + res.records_stored) * res.slot_bytes
            rec["kernel_ms"] += res.kernel_ms
            rec["launches"] += 1
        return out

    _eng.run_search = run_search_probe

    clk = ClockSampler(device).__enter__()  # running before the timed region
    for _ in range(args.warmup):
        pair(g)
    barrier()
    rec.update(bytes=0, kernel_ms=0.0, launches=0)
    l0 = _lib.launch_count()
    total_ms, nodes = 0.0, 0.0
    clk.mark_start()
    for _ in range(args.steps):
        flush.zero_()  # L2 flush between timed steps (outside the events)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        nd, _ = pair(g)
        e1.record()
        torch.cuda.synchronize()
        total_ms += e0.elapsed_time(e1)
        nodes += nd
    clk.mark_end()
    clk.__exit__(None, None, None)
    launches = _lib.launch_count() - l0
    search_bytes, search_ms, search_launches = rec["bytes"], rec["kernel_ms"], rec["launches"]

    # e2e: from host numpy buffers every step (upload + solve + readback)
    h2d = (n + 1) * 4 + len(nbr) * 4
    e2e_ms, e2e_nodes = 0.0, 0.0
    for _ in range(args.steps):
        flush.zero_()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gh = vc.StaticGraph(n, np.array(off), np.array(nbr))
        nd, _ = pair(gh)
        e1.record()
        torch.cuda.synchronize()
        e2e_ms += e0.elapsed_time(e1)
        e2e_nodes += nd
    # per solve the host reads back the reduced CSR + vertex map + forced ids
    # (int32), the components histogram (int64) and the result structs
    rg = vc.root_reduce(g, bound=opt).graph
    d2h = 2 * ((rg.num_vertices + 1) * 4 + len(rg.neighbors) * 4 + rg.num_vertices * 4
               + n * 4 + (rg.num_vertices + 2) * 8 + 512)

    t = torch.tensor([total_ms, nodes, e2e_ms, e2e_nodes], dtype=torch.float64,
                     device="cuda" if world <= ndev else "cpu")
    if world > 1:
        tmax = t.clone()
        torch.distributed.all_reduce(tmax, op=torch.distributed.ReduceOp.MAX)
        tsum = t.clone()
        torch.distributed.all_reduce(tsum, op=torch.distributed.ReduceOp.SUM)
        total_ms, e2e_ms = float(tmax[0]), float(tmax[2])
        if strong:  # solve_distributed already reports whole-job node counts
            nodes, e2e_nodes = float(t[1]), float(t[3])
        else:
            nodes, e2e_nodes = float(tsum[1]), float(tsum[3])
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
    peak = peaks.get("hbm_gbs") or 6650.0
    peak_src = "measured" if peaks.get("hbm_gbs") else "fallback"
    per_launch_bytes = search_bytes / max(search_launches, 1)
    per_launch_ms = search_ms / max(search_launches, 1)
    achieved = per_launch_bytes / (per_launch_ms * 1e-3) / 1e9 if per_launch_ms else 0.0
    traffic, _ = load_traffic()
    line = {
        "metric": METRIC,
        "value": nodes / (total_ms * 1e-3),
        "unit": "nodes/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps,
        "time_to_solution_s": total_ms / args.steps * 1e-3,
        "higher_is_better": True,
        "scaling": "strong" if strong else "weak",
        "vs_baseline": None,
        "dtype": "int32",
        "data": "synthetic (seeded random geometric graph, seed 1)" if strong else
                "synthetic (seeded random geometric graph, seed 1 + rank)",
        "config": {"workload": WORKLOAD, "opt": opt, "n": n, "m": len(nbr) // 2,
                   "parallelism": (f"{world} GPUs on one instance (root-subtree partition, "
                                   "NCCL MIN all-reduce of the bound)") if strong else
                                  f"dp{world} (independent instances)",
                   "l2": "flushed between timed steps (512 MiB write)"},
        "e2e": {"value": e2e_nodes / (e2e_ms * 1e-3), "unit": "nodes/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_ms / args.steps},
        "gpu_launches": launches,
        "roofline": {
            "bound": "hbm", "kernel": "search_kernel", "achieved": achieved, "peak": peak,
            "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic,
            "algorithmic_bytes_per_launch": per_launch_bytes,
            "launch_ms": per_launch_ms,
            # summed over the step's two concurrent searches: may exceed 1
            "kernel_share_of_step": search_ms / total_ms if total_ms else None,
        },
        "clocks": clk.summary(),
    }
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

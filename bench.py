"""Benchmark of the CJM hot path (BASELINE.json metric: GLUPS and time-to-tol
vs the HBM roofline).

    python bench.py [--gpus N --steps K --warmup W] [--config NAME] [--impl cjm|reference]

A step is one pass of the whole hot path:
cjm_plan (bounds, cycle length, ordering, weights -> device) + cjm_solve to
tolerance (setup, every sweep, the fused residual checks, the stop decision)
+ cjm_plan_destroy, on the paper's test problem, inputs resident
in HBM.  value = nx * ny * iterations (all ranks) / step time = GLUPS.

Default workload: BASELINE.json configs[2], the 9-point stencil at 4096^2 on
one B200 ("single-GPU roofline config"; three 134 MB arrays, larger than L2,
so every sweep streams from HBM).  Under torchrun with N GPUs the grid grows
with N (weak scaling, row slabs of 4096 x 4096 per GPU, NCCL halo exchange).

The reference arm (--impl reference) is the CPU oracle (there is no reference
code, only the paper): a bounded segment of the same solve on the host cores.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_LUP = 24          # read u, read g, write u'
CONFIGS = {
    # name: (stencil, nx, ny_per_gpu, tol, BASELINE.json config)
    "cjm9_4096": (9, 4096, 4096, 1e-8, "configs[2]: 9-point CJM at 4096^2 on 1 B200"),
    "cjm9_16384": (9, 16384, 16384, 1e-8, "north_star target: 9-point CJM at 16384^2"),
    "cjm17_8192": (17, 8192, 8192, 1e-8, "configs[3]: 17-point at 8192^2"),
    "cjm9_1024": (9, 1024, 1024, 1e-8, "configs[1]: 9-point at 1024^2"),
    "cjm5_1024": (5, 1024, 1024, 1e-8, "configs[1]: 5-point at 1024^2"),
    "cjm17_1024": (17, 1024, 1024, 1e-8, "17-point at 1024^2 (tab:tab01 size)"),
    "cjm9_64": (9, 64, 64, 1e-8, "configs[0]: 9-point at 64^2"),
    # configs[4]: 9-point at 32768 columns; weak = 4096-row slab per GPU (ny = 4096 G),
    # strong = the whole 32768^2 grid (one GPU holds it: 3 x 8.6 GB; ~4 min per solve)
    "cjm9_32768w": (9, 32768, 4096, 1e-8, "configs[4] weak: 9-point, 32768 x 4096 slab per GPU"),
    "cjm9_32768": (9, 32768, 32768, 1e-8, "configs[4] strong: 9-point at 32768^2"),
}
METRIC = "GLUPS (fp64 lattice updates/s) and time-to-tol vs HBM roofline"


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def ncu_traffic(config):
    """Per-launch DRAM bytes of the sweep kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "sweep_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    v = d.get(config)
    return None if v is None else float(v["dram_bytes_per_launch"])


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4)
                          if len(s) > 2 + k and s[2 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def make_problem(stencil, nx, ny, y0, nyl):
    """Global test problem rows [y0, y0+nyl) (+ ghosts) of the weak-scaled grid."""
    from paper_1705_00103_b200 import inputs
    from paper_1705_00103_b200.cjm import cjm_schedule  # noqa: F401  (library must load)
    r = 2 if stencil == 17 else 1
    h = inputs.grid_h(nx, ny)
    xg = inputs.coords(nx, r, h)
    yg = (np.arange(y0 + 1 - r, y0 + nyl + r + 1, dtype=np.float64)) * h
    u0 = inputs.exact(xg, yg)
    u0[r:r + nyl, r:r + nx] = 0.0
    b = inputs.source(xg[r:r + nx], yg[r:r + nyl])
    return np.ascontiguousarray(u0), np.ascontiguousarray(b), h


def cpu_oracle_glups(stencil, nx, ny, h, budget_s):
    """The oracle as it stands, on a bounded segment of the same solve
    (full-size grid, first sweeps of the schedule), on all host cores."""
    import oracle
    from paper_1705_00103_b200 import inputs
    r = oracle.reach(stencil)
    u0, b, _ = inputs.test_problem(nx, ny, r, h=h)
    s = oracle.schedule(stencil, nx, ny, 1e-8)
    g = oracle.rhs_to_g(stencil, h, b)
    # calibrate (doubling until 0.5 s), then one oracle call of k sweeps lasting ~budget_s
    c = 1
    while True:
        t0 = time.perf_counter()
        oracle.sweeps(stencil, u0, g, s["w"], 0, c)
        per = (time.perf_counter() - t0) / c
        if per * c >= 0.5 or c >= 4096:
            break
        c *= 2
    k = max(2, int(budget_s / max(per, 1e-9)))
    t0 = time.perf_counter()
    oracle.sweeps(stencil, u0, g, s["w"], 0, k)
    dt = time.perf_counter() - t0
    return dict(value=k * nx * ny / dt / 1e9, unit="GLUPS", cores=oracle.num_threads(),
                kind="oracle", sample=f"{k} sweeps of the {stencil}-point {nx}x{ny} solve "
                f"(schedule positions 0..{k - 1}), {dt:.1f} s, OpenMP over rows")


def run_reference(args, rank, world):
    if rank != 0:
        return
    stencil, nx, nyg, tol, desc = CONFIGS[args.config]
    import oracle
    from paper_1705_00103_b200 import inputs
    # torchrun exports OMP_NUM_THREADS=1 to every rank; rank 0 alone works
    # here, so it takes all host cores the process may run on
    oracle.set_num_threads(len(os.sched_getaffinity(0)))
    h = inputs.grid_h(nx, nyg)
    steps = []
    for _ in range(args.warmup + args.steps):
        steps.append(cpu_oracle_glups(stencil, nx, nyg, h, budget_s=args.ref_seconds))
    timed = steps[args.warmup:]
    val = statistics.median([s["value"] for s in timed])
    cb = dict(timed[-1])
    cb["value"] = val
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "GLUPS", "n_gpus": world,
            "working_ranks": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * args.ref_seconds, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "stencil": stencil, "nx": nx, "ny": nyg,
                       "tol": tol, "baseline_config": desc},
            "cpu_baseline": cb,
            "e2e": {"value": val, "unit": "GLUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cjm", choices=["cjm", "reference"])
    ap.add_argument("--config", default="cjm9_4096", choices=sorted(CONFIGS))
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--tile-w", type=int, default=0)
    ap.add_argument("--stages", type=int, default=0)
    ap.add_argument("--ctas-per-sm", type=int, default=0)
    ap.add_argument("--graph-chunk", type=int, default=0)
    ap.add_argument("--temporal-k", type=int, default=0)
    args = ap.parse_args()

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local_rank = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_1705_00103_b200 import cjm

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    stencil, nx, ny_per, tol, desc = CONFIGS[args.config]
    ny = ny_per * world
    y0, nyl = cjm.cjm_slab(ny, world, rank)
    u0, b, h = make_problem(stencil, nx, ny, y0, nyl)
    nccl_id = None
    if world > 1:
        idt = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(cjm.cjm_get_nccl_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        nccl_id = bytes(idt.cpu().numpy().tobytes())
    opts = dict(device=local_rank, world_size=world, rank=rank, tile_w=args.tile_w,
                stages=args.stages, ctas_per_sm=args.ctas_per_sm, graph_chunk=args.graph_chunk,
                temporal_k=args.temporal_k)
    stream = torch.cuda.current_stream()
    u_dev0 = torch.from_numpy(u0).to(dev)
    b_dev = torch.from_numpy(b).to(dev)
    u_dev = torch.empty_like(u_dev0)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local_rank])
        torch.cuda.synchronize()

    def step(host=False, uh=None, bh=None):
        plan = cjm.Plan(stencil, nx, ny, h, tol, nccl_id=nccl_id, **opts)
        try:
            if host:
                rep = plan.solve_host(bh, uh, stream)
            else:
                u_dev.copy_(u_dev0)  # restore u_0 (device-to-device, outside the solve's bytes)
                rep = plan.solve(b_dev, u_dev, stream)
        finally:
            plan.close()
        return rep

    def timed(n, host=False):
        reps = []
        bh, uhs = None, [None] * n
        if host:   # one pinned copy of u_0 per step, filled before the timed region
            bh = torch.from_numpy(b).pin_memory()
            uhs = [torch.from_numpy(u0).pin_memory() for _ in range(n)]
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        ev0.record(stream)
        for k in range(n):
            reps.append(step(host, uhs[k], bh))
        ev1.record(stream)
        barrier()
        t = ev0.elapsed_time(ev1) / 1e3
        tt = torch.tensor([t], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item()), reps

    for _ in range(args.warmup):
        step()
    with ClockSampler(local_rank) as clk:
        t_dev, reps = timed(args.steps)
    clocks = clk.summary()
    iters = reps[-1]["iterations"]
    lups_total = float(nx) * ny * sum(r["iterations"] for r in reps)
    value = lups_total / t_dev / 1e9
    # dominant kernel: the hot sweep kernel (K fused sweeps per launch), timed
    # with CUDA events on its launching stream around the graph launches
    sweep_s = sum(r["sweep_s"] for r in reps)
    hot = sum(r["hot_launches"] for r in reps)
    K = reps[-1]["temporal_k"]
    t_launch = sweep_s / max(hot, 1)
    bytes_per_launch = BYTES_PER_LUP * float(nx) * nyl      # read u, read g, write u' once per launch
    achieved = bytes_per_launch / t_launch / 1e9
    peak, peak_kind = measured_peaks()
    traffic = ncu_traffic(args.config) if world == 1 else None
    launches = int(sum(r["kernel_launches"] for r in reps))

    e2e = None
    if not args.no_e2e:
        step(host=True, uh=torch.from_numpy(u0.copy()).pin_memory(),
             bh=torch.from_numpy(b).pin_memory())
        t_e2e, reps_h = timed(args.steps, host=True)
        e2e = {"value": float(nx) * ny * sum(r["iterations"] for r in reps_h) / t_e2e / 1e9,
               "unit": "GLUPS",
               "h2d_bytes_per_step": int(reps_h[-1]["h2d_bytes"]) * world,
               "d2h_bytes_per_step": int(reps_h[-1]["d2h_bytes"]) * world,
               "ms_per_step": 1e3 * t_e2e / args.steps,
               "api": "cjm_solve_host (pinned host buffers)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_oracle_glups(stencil, nx, ny, h, budget_s=args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GLUPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_dev / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": args.config, "stencil": stencil, "nx": nx, "ny": ny,
                       "ny_per_gpu": ny_per, "tol": tol, "baseline_config": desc,
                       "parallelism": f"row-slab x{world}" if world > 1 else "single GPU",
                       "l2": "inputs larger than L2 (3 x %.0f MB per GPU vs 126 MB L2)"
                             % (nx * ny_per * 8 / 1e6),
                       "step": "cjm_plan + cjm_solve to tol + cjm_plan_destroy"},
            "time_to_tol_s": t_dev / args.steps, "iterations": iters,
            "cycles": reps[-1]["cycles"], "cycle_len": reps[-1]["cycle_len"],
            "r_ratio": reps[-1]["r_l2"] / reps[-1]["r0_l2"],
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_source": f"{peak_kind} copy bandwidth (MEASURED_PEAKS.json hbm_gbs)",
                         "kernel": f"cjm_sweep_kernel<{stencil},K={K}>",
                         "sweeps_per_launch": K,
                         "algorithmic_bytes_per_launch": bytes_per_launch,
                         "avg_launch_us": 1e6 * t_launch,
                         "sweep_glups": K * float(nx) * nyl / t_launch / 1e9,
                         # the same launches against the single-sweep roofline
                         # (24 B per lattice update): > 1 because a
                         # launch moves 24 B per node for K updates
                         "lup_roofline_frac": K * float(nx) * nyl / t_launch * BYTES_PER_LUP
                                              / 1e9 / peak,
                         "note": (f"{K} sweeps per launch share one pass over HBM (24 B per node "
                                  "per launch); with K > 1 the launch is fp64-latency bound, not "
                                  "HBM bound (DESIGN section 5)") if K > 1 else None},
            "breakdown_ms": {"plan": 1e3 * statistics.mean(r["plan_s"] for r in reps),
                             "solve_device": 1e3 * statistics.mean(r["solve_s"] for r in reps),
                             "hot_sweeps": 1e3 * statistics.mean(r["sweep_s"] for r in reps)},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

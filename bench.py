"""Benchmark of the CJM hot path (BASELINE.json metric: GLUPS and time-to-tol
vs the HBM roofline at 1/2/4/8 B200).

    python bench.py [--gpus N --steps K --warmup W] [--config NAME] [--impl cjm|reference]

A step is one pass of the whole hot path:
cjm_plan (bounds, cycle length, ordering, weights -> device) + cjm_solve to
tolerance (setup, every sweep, the fused residual checks, the stop decision)
+ cjm_plan_destroy, on the paper's test problem, inputs resident
in HBM.  value = nx * ny * iterations / step time = GLUPS (whole job).

Default workload: the north_star target, the 9-point stencil at 16384^2
(three 2.1 GB arrays per GPU, far larger than the 126 MB L2, so every launch
streams from HBM).  Under torchrun with N GPUs the SAME grid is split into N
row slabs (strong scaling, NCCL halo exchange; N = 1 is the single-GPU line).
configs[4]'s weak slab (`--config cjm9_32768w`: 32768 x 4096 rows per GPU)
is the weak-scaling variant.

The reference arm (--impl reference) is the CPU oracle (there is no reference
code, only the paper): each step a bounded segment of the same solve on the
host cores, rank 0 only.
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
# fp64 pipe operations (DADD + DFMA) per lattice update of the fixed
# association of DESIGN R6, pair sums shared between rows: 5-point 4 DADD +
# 2 DFMA, 9-point 5 + 3, 17-point 8 + 6
FP64_OPS_PER_LUP = {5: 6, 9: 8, 17: 14}
CONFIGS = {
    # name: (stencil, nx, ny, tol, scaling, BASELINE.json config)
    #   strong: ny is the global grid (split into N slabs); weak: ny rows per GPU
    "cjm9_16384": (9, 16384, 16384, 1e-8, "strong", "north_star target: 9-point CJM at 16384^2"),
    "cjm9_4096": (9, 4096, 4096, 1e-8, "strong", "configs[2]: 9-point CJM at 4096^2 on 1 B200"),
    "cjm17_8192": (17, 8192, 8192, 1e-8, "strong", "configs[3]: 17-point at 8192^2"),
    "cjm9_1024": (9, 1024, 1024, 1e-8, "strong", "configs[1]: 9-point at 1024^2"),
    "cjm5_1024": (5, 1024, 1024, 1e-8, "strong", "configs[1]: 5-point at 1024^2"),
    "cjm17_1024": (17, 1024, 1024, 1e-8, "strong", "17-point at 1024^2 (tab:tab01 size)"),
    "cjm9_64": (9, 64, 64, 1e-8, "strong", "configs[0]: 9-point at 64^2"),
    "cjm9_32768": (9, 32768, 32768, 1e-8, "strong", "configs[4] strong: 9-point at 32768^2"),
    "cjm9_32768w": (9, 32768, 4096, 1e-8, "weak", "configs[4] weak: 9-point, 32768 x 4096 slab per GPU"),
}
DEFAULT_CONFIG = "cjm9_16384"
METRIC = "GLUPS (fp64 lattice updates/s) and time-to-tol vs HBM roofline"
DIGESTS = os.path.join(ROOT, "tests", "golden", "oracle_digests.json")


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def grid(config, world):
    stencil, nx, ny, tol, scaling, desc = CONFIGS[config]
    return stencil, nx, (ny * world if scaling == "weak" else ny), tol, scaling, desc


def config_dict(config, world):
    """The `config` object of both arms' JSON lines (identical by construction)."""
    stencil, nx, ny, tol, scaling, desc = grid(config, world)
    return {"workload": config, "stencil": stencil, "nx": nx, "ny": ny, "tol": tol,
            "baseline_config": desc,
            "parallelism": f"row-slab x{world}" if world > 1 else "single GPU",
            "l2": "inputs larger than L2 (3 x %.0f MB per GPU vs 126 MB L2)"
                  % (nx * (ny // world) * 8 / 1e6),
            "step": "cjm_plan + cjm_solve to tol + cjm_plan_destroy"}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def fp64_peak():
    """Measured fp64 pipe peak (DFMA lane-operations/s, profiles/fp64_peak.json,
    scripts/fp64_peak.cu run on a B200)."""
    p = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if not os.path.exists(p):
        return None, None
    with open(p) as f:
        d = json.load(f)
    return float(d["dfma_ops_per_s"]), d.get("how", "")


def ncu_traffic(config):
    """Per-launch DRAM bytes of the sweep kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "sweep_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    v = d.get(config)
    return None if v is None else float(v["dram_bytes_per_launch"])


def oracle_iterations(config):
    """The oracle's stored iteration count of this config's full solve, if any
    (tests/golden/oracle_digests.json, written by tests/make_oracle_digests.py)."""
    if not os.path.exists(DIGESTS):
        return None
    with open(DIGESTS) as f:
        rec = json.load(f).get(config)
    return None if rec is None else int(rec["report"]["iterations"])


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw")

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
        pw = []
        for s in self.samples:
            try:
                pw.append(float(s[6]))
            except (IndexError, ValueError):
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "power_w": statistics.median(pw) if pw else None,
                "samples": len(self.samples)}


def make_problem(stencil, nx, ny, y0, nyl):
    """Global test problem rows [y0, y0+nyl) (+ ghosts) of the nx x ny grid."""
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


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


class OracleSample:
    """The oracle as it stands on a bounded segment of the same solve
    (full-size grid, the first sweeps of the schedule), all host cores.  The
    inputs are generated once; each run() times one oracle call of k sweeps."""

    def __init__(self, stencil, nx, ny):
        import oracle
        from paper_1705_00103_b200 import inputs
        self.oracle = oracle
        self.stencil, self.nx, self.ny = stencil, nx, ny
        r = oracle.reach(stencil)
        h = inputs.grid_h(nx, ny)
        self.u0, b, _ = inputs.test_problem(nx, ny, r, h=h)
        self.s = oracle.schedule(stencil, nx, ny, 1e-8)
        self.g = oracle.rhs_to_g(stencil, h, b)
        self.k = None

    def calibrate(self, budget_s):
        """Sweeps per call so that one call lasts ~budget_s.  The per-sweep
        cost is the marginal one (two calls of c and 3c sweeps, c doubled until
        the longer call lasts >= 0.5 s): each oracle call also pays a fixed
        cost (a second full-size buffer), which a long call amortises."""
        c = 1
        while True:
            t0 = time.perf_counter()
            self.oracle.sweeps(self.stencil, self.u0, self.g, self.s["w"], 0, c)
            t1 = time.perf_counter()
            self.oracle.sweeps(self.stencil, self.u0, self.g, self.s["w"], 0, 3 * c)
            t3 = time.perf_counter() - t1
            t1 -= t0
            if t3 >= 0.5 or c >= 4096:
                break
            c *= 2
        per = max((t3 - t1) / (2 * c), t3 / (3 * c) * 0.25, 1e-9)
        fixed = max(t1 - per * c, 0.0)
        self.k = max(2, int((budget_s - fixed) / per))
        return self.k

    def run(self):
        t0 = time.perf_counter()
        self.oracle.sweeps(self.stencil, self.u0, self.g, self.s["w"], 0, self.k)
        dt = time.perf_counter() - t0
        return self.k * self.nx * self.ny / dt / 1e9, dt

    def describe(self, dt, glups, iters):
        d = dict(value=glups, unit="GLUPS", cores=self.oracle.num_threads(), kind="oracle",
                 cpu_model=cpu_model(),
                 sample=f"{self.k} sweeps of the {self.stencil}-point {self.nx}x{self.ny} solve "
                        f"(schedule positions 0..{self.k - 1}), {dt:.1f} s, OpenMP over rows")
        if iters:
            d["time_to_tol_extrapolated_s"] = iters * self.nx * self.ny / (glups * 1e9)
            d["iterations_to_tol"] = iters
        return d


def run_reference(args, rank, world):
    if rank != 0:
        return
    stencil, nx, ny, tol, scaling, desc = grid(args.config, world)
    import oracle
    # torchrun exports OMP_NUM_THREADS=1 to every rank; rank 0 alone works
    # here, so it takes all host cores the process may run on
    oracle.set_num_threads(len(os.sched_getaffinity(0)))
    smp = OracleSample(stencil, nx, ny)
    smp.calibrate(args.ref_seconds)
    for _ in range(args.warmup):
        smp.run()
    timed = [smp.run() for _ in range(args.steps)]
    val = statistics.median(g for g, _ in timed)
    step_s = statistics.mean(dt for _, dt in timed)
    iters = oracle_iterations(args.config) or smp.s["P"]
    cb = smp.describe(step_s, val, iters)
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "GLUPS", "n_gpus": world,
            "working_ranks": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * step_s, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(args.config, world),
            "cpu_baseline": cb,
            "e2e": {"value": val, "unit": "GLUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cjm", choices=["cjm", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-seconds", type=float, default=6.0)
    ap.add_argument("--e2e-steps", type=int, default=5, help="timed e2e steps (<= --steps)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--tile-w", type=int, default=0)
    ap.add_argument("--stages", type=int, default=0)
    ap.add_argument("--ctas-per-sm", type=int, default=0)
    ap.add_argument("--graph-chunk", type=int, default=0)
    ap.add_argument("--temporal-k", type=int, default=0)
    ap.add_argument("--warps", type=int, default=0)
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
    stencil, nx, ny, tol, scaling, desc = grid(args.config, world)
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
                temporal_k=args.temporal_k, warps=args.warps)
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

    def max_over_ranks(t):
        tt = torch.tensor([t], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    for k in range(args.warmup):
        rep0 = step()
        if k == 0 and world > 1:
            # one line per rank (stderr): the NCCL communicator the plan runs on
            print(json.dumps({"rank": rank, "world_size": world, "comm_nranks": rep0["comm_nranks"],
                              "comm_rank": rep0["comm_rank"], "slab": [y0, nyl],
                              "temporal_k": rep0["temporal_k"], "warps": rep0["warps"],
                              "ctas": rep0["ctas"]}), file=sys.stderr, flush=True)

    # ---- device-resident timed region: EXACTLY args.steps steps
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        barrier()
        ev0.record(stream)
        reps = [step() for _ in range(args.steps)]
        ev1.record(stream)
        barrier()
    t_dev = max_over_ranks(ev0.elapsed_time(ev1) / 1e3)
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
    f64_peak, f64_how = fp64_peak()
    fp64_achieved = FP64_OPS_PER_LUP[stencil] * K * float(nx) * nyl / t_launch

    # ---- end to end through cjm_solve_host: one pinned u / rhs buffer, u
    # refreshed from u_0 OUTSIDE each step's timed region
    e2e = None
    if not args.no_e2e:
        bh = torch.from_numpy(b).pin_memory()
        uh = torch.from_numpy(u0.copy()).pin_memory()
        uh_np = uh.numpy()
        step(host=True, uh=uh, bh=bh)
        n_e2e = max(1, min(args.steps, args.e2e_steps))
        t_e2e, reps_h = 0.0, []
        for _ in range(n_e2e):
            np.copyto(uh_np, u0)
            barrier()
            ev0.record(stream)
            reps_h.append(step(host=True, uh=uh, bh=bh))
            ev1.record(stream)
            barrier()
            t_e2e += ev0.elapsed_time(ev1) / 1e3
        t_e2e = max_over_ranks(t_e2e)
        e2e = {"value": float(nx) * ny * sum(r["iterations"] for r in reps_h) / t_e2e / 1e9,
               "unit": "GLUPS",
               "h2d_bytes_per_step": int(reps_h[-1]["h2d_bytes"]) * world,
               "d2h_bytes_per_step": int(reps_h[-1]["d2h_bytes"]) * world,
               "ms_per_step": 1e3 * t_e2e / n_e2e, "steps": n_e2e,
               "api": "cjm_solve_host (pinned host buffers; u refreshed outside the timed region)"}
        del bh, uh

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        smp = OracleSample(stencil, nx, ny)
        smp.calibrate(args.cpu_seconds)
        g_cpu, dt = smp.run()
        cpu = smp.describe(dt, g_cpu, oracle_iterations(args.config) or iters)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GLUPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_dev / args.steps,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": config_dict(args.config, world),
            "time_to_tol_s": t_dev / args.steps, "iterations": iters,
            "oracle_iterations": oracle_iterations(args.config),
            "cycles": reps[-1]["cycles"], "cycle_len": reps[-1]["cycle_len"],
            "r_ratio": reps[-1]["r_l2"] / reps[-1]["r0_l2"],
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_source": f"{peak_kind} copy bandwidth (MEASURED_PEAKS.json hbm_gbs)",
                         "kernel": f"cjm_sweep_kernel_v4<{stencil},NW={reps[-1]['warps']},K={K}>",
                         "sweeps_per_launch": K,
                         "algorithmic_bytes_per_launch": bytes_per_launch,
                         "avg_launch_us": 1e6 * t_launch,
                         "sweep_glups": K * float(nx) * nyl / t_launch / 1e9,
                         # the same launches against the single-sweep roofline
                         # (24 B per lattice update): > 1 because a
                         # launch moves 24 B per node for K updates
                         "lup_roofline_frac": K * float(nx) * nyl / t_launch * BYTES_PER_LUP
                                              / 1e9 / peak,
                         # the fp64 pipe: FP64_OPS_PER_LUP DADD/DFMA per update
                         # against the measured DFMA issue peak
                         "fp64_ops_per_lup": FP64_OPS_PER_LUP[stencil],
                         "fp64_frac": fp64_achieved / f64_peak if f64_peak else None,
                         "fp64_peak_ops_per_s": f64_peak,
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

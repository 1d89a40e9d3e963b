#!/usr/bin/env python
"""bench.py — swept 1-D heat (FTCS, FP64) on B200, the BASELINE.json headline.

Metric: BASELINE.json `metric` (point-updates/s, swept vs classic), on the
configuration it is quoted on that fits one GPU: configs[1] = heat FP64,
n = 2^27 per GPU, block width 1024 (the block-size sweep 32–1024 puts w = 256,
512 and 1024 within 0.5% of each other at this n, profiles/r02j_heat_report.txt;
at the bench's T, w = 1024 is the fastest both on the device, 2.874 vs 2.863 T,
and end to end, 2.79 vs 2.74 T — the reference's best-config reporting),
T = 6144 time steps per run (the paper's ~6000, a multiple of
every m = w/2 <= 512 so no classic pad is timed).

One bench "step" = one full solve (`s1d_advance`: UpTriangle, Diamonds,
DownTriangle) of T time steps from the resident initial condition. `value` is
device-timed (CUDA events inside the library, on the launching streams), the
max over ranks; `e2e` times the same solve through the C ABI with pinned HOST
buffers (H2D of the IC, solve, D2H of the state) every step; the library
overlaps those copies with the first and last phases of the solve, chunk by
chunk ("wavefront solve").

--impl reference runs the reference's own CPU engine (sweep1d::run, swept,
WallClock, compiled from source into oracle/_ref) on this host's cores on a
bounded sample of the same workload.

Multi-GPU (torchrun, one process per GPU): weak scaling, n = 2^27 per GPU;
see DESIGN.md "Multi-GPU".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("Mpt-updates/s (heat, Euler Sod) swept vs classic at 1/2/4/8 B200; µs/timestep")
UNIT = "Mpt-updates/s"
HEAT_FLOPS_PER_UPDATE = 5  # heat_step: 2 mul + 3 add (inc/kernels.hpp:14-16)
# FP64-pipe instructions per point-update the tile kernels need under bitwise
# parity: l - 2c as one fma (2c is exact; heat.cu heat_step), then the three
# separately rounded add, mul, add. The fast form runs at this config (Fo =
# 0.4, |T| <= 1); the exact form needs 5.
HEAT_FP64_INSTR_PER_UPDATE = 4
CLASSIC_BYTES_PER_UPDATE = 16  # one FP64 load + one store per point-update


def euler_pipe_profile():
    """FP64-pipe utilisation of the Euler swept Diamond (both methods) from the
    committed ncu capture of this configuration (profiles/r02_euler_top_kernel.txt):
    the Euler kernels are FP64-pipe bound (div/sqrt-heavy fluxes)."""
    path = os.path.join(ROOT, "profiles", "r02_euler_top_kernel.txt")
    out = {"bound": "fp64", "kernel": "euler_tile (swept Diamond)", "unit": "% of FP64 pipe cycles",
           "source": "ncu sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active, " + os.path.relpath(path, ROOT)}
    try:
        method = None
        for line in open(path):
            if line.startswith("== ") and "euler_tile<" in line:
                method = "flattening" if "euler_tile<1" in line else "lengthening"
            elif method and "sm__pipe_fp64_cycles_active" in line:
                out[f"{method}_fp64_pipe_active_pct"] = float(line.split()[1])
    except OSError:
        return None
    return out


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_dev{device}.csv")

    def __enter__(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.fh,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        with open(self.path) as fh:
            for line in fh:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 8:
                    rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        loaded = [s for s in sm if s > 0.5 * (max(smax) if smax else 0)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(rows)}


def dist_init():
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method="env://")
    return rank, world


def relaunch_under_torchrun(argv, n):
    """`python bench.py --gpus N` outside a launcher: re-exec this script under
    torch.distributed.run with N processes (one per GPU), the same launch the
    driver uses; the JSON line comes from rank 0 of that job."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + list(argv)
    sys.stdout.flush()
    sys.stderr.flush()
    os.execv(sys.executable, cmd)


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def ring_connect_record(rank, world, local, shard):
    """After the shards are connected: one line per rank on stderr with the
    ring it joined (the data plane is peer-pointer reads over NVLink, not a
    NCCL collective), and - when every rank has its own GPU - a NCCL
    communicator over the same ranks, checked with one all-reduce, so the job's
    GPU set is visible to NCCL_DEBUG as well. Returns rank 0's summary."""
    import torch
    import torch.distributed as dist
    start, count = shard.start, shard.count
    left, right = (rank + world - 1) % world, (rank + 1) % world
    nccl_ok = None
    if torch.cuda.is_available() and world <= torch.cuda.device_count():
        try:
            torch.cuda.set_device(local)
            g = dist.new_group(backend="nccl")
            t = torch.ones(1, device=f"cuda:{local}")
            dist.all_reduce(t, group=g)
            torch.cuda.synchronize(local)
            nccl_ok = int(t.item()) == world
        except Exception as ex:  # reported, the data plane does not depend on it
            nccl_ok = f"nccl group unavailable: {ex!r}"[:200]
    print(f"[bench] ring connect: rank {rank} nranks {world} cudaDev {local} left {left} right {right} "
          f"shard [{start}, {start + count}) nccl_allreduce_ok {nccl_ok}", file=sys.stderr, flush=True)
    recs = [None] * world
    dist.all_gather_object(recs, {"rank": rank, "device": local, "start": start, "count": count})
    return {"nranks": world, "devices": [r["device"] for r in recs],
            "shards": [[r["start"], r["count"]] for r in recs], "nccl_allreduce_ok": nccl_ok,
            "transport": "peer-pointer edge reads over NVLink (CUDA IPC) + device flags, one message per "
                         "shard per half-cycle"}


def allmax(world, x: float) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# --------------------------------------------------------------------------
# CPU reference (oracle/_ref: the reference compiled from source)
# --------------------------------------------------------------------------
def divisor_ranks(blocks: int, want: int) -> int:
    for r in range(max(want, 1), 0, -1):
        if blocks % r == 0:
            return r
    return 1


def cpu_reference_sample(equation, scheme, w, n_sample, steps, threads):
    """One run of the reference's own engine (sweep1d::run, compiled from
    source into oracle/_ref) with one rank thread per host core (the reference
    runs R rank threads, engines_impl.hpp:35-67; R must divide the block count
    and be >= 2, config.cpp:79-81)."""
    from oracle import oracle as O
    blocks = n_sample // w
    ranks = max(divisor_ranks(blocks, threads), 2)
    cfg = O.RefConfig(equation=equation, scheme=scheme, grid_size=n_sample, block_width=w, ranks=ranks,
                      steps=steps, mode="wall")
    res = O.ref_run(cfg)
    rate = n_sample * steps / res.loop_seconds
    return rate, ranks, res.loop_seconds


def reference_sample_size(args, timed_steps):
    """The reference arm's per-step sample: the B200 arm's grid (n = 2^log2n,
    same w) for T = m = w/2 time steps (one swept cycle: Up + Down, no classic
    pad; T < m would be all pad, swept_worker :313-320). Only T differs from
    the GPU arm. If `timed_steps` of it would overrun --ref-budget-s (measured
    rate from a small calibration run), n is halved until it fits, and the
    line says so."""
    m = args.w // 2
    steps = args.ref_steps or m
    steps = max(m, (steps // m) * m)
    n = args.ref_n or (1 << args.log2n)
    rate, _, _ = cpu_reference_sample(args.equation, args.scheme, args.w, min(n, 1 << 22), m, host_cores())
    while n > args.w * 64 and timed_steps * n * steps / rate > args.ref_budget_s:
        n //= 2
    return n, steps, rate


def run_reference_arm(args, rank, world):
    if rank != 0:
        return 0  # the CPU reference runs once, on rank 0 (the host's cores are shared)
    threads = host_cores()
    w = args.w
    t_all = time.perf_counter()
    n_sample, steps_sample, _ = reference_sample_size(args, args.steps)
    vals, ranks = [], 0
    for i in range(args.warmup + args.steps):
        # warm-up steps run a small sample (untimed); timed steps the full one
        n_i = n_sample if i >= args.warmup else min(n_sample, 1 << 22)
        rate, ranks, secs = cpu_reference_sample(args.equation, args.scheme, w, n_i, steps_sample, threads)
        if i >= args.warmup:
            vals.append(rate)
    value = statistics.mean(vals) / 1e6
    same_n = n_sample == (1 << args.log2n)
    sample = (f"sweep1d::run({args.scheme}, WallClock) {args.equation} n=2^{n_sample.bit_length() - 1} w={w} "
              f"T={steps_sample} per step, {ranks} rank threads on {threads} host cores"
              + ("; only T differs from the GPU arm (T = m: one swept cycle, no pad)" if same_n else
                 f"; n reduced from 2^{args.log2n} to fit --ref-budget-s {args.ref_budget_s:g}")
              + (f"; rank 0 of {world}, per-point throughput (the host's cores do not grow with N)"
                 if world > 1 else ""))
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * n_sample * steps_sample / (value * 1e6), 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (heat-sine IC)",
        "config": {"workload": workload_name(args), "equation": args.equation, "scheme": args.scheme,
                   "grid_size": n_sample, "block_width": w, "steps_per_run": steps_sample,
                   "same_config_except_T": same_n},
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": ranks, "kind": "reference",
                         "host_cores": threads, "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_seconds": round(time.perf_counter() - t_all, 2),
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_name(args):
    return (f"{args.equation} {args.scheme} FP64, n=2^{args.log2n} per GPU, block width {args.w}, "
            f"T={args.T} time steps per run (BASELINE configs[1]/[3])")


# --------------------------------------------------------------------------
# B200 arm
# --------------------------------------------------------------------------
def run_b200(args, rank, world):
    import numpy as np
    import paper_1811_08282_b200 as s1d

    if s1d.device_count() == 0:
        raise SystemExit("bench.py: no CUDA device visible (the B200 path has no CPU fallback)")
    local = env_int("LOCAL_RANK", 0) % s1d.device_count()  # this rank's GPU
    n_per = 1 << args.log2n
    eq = s1d.Equation.Heat if args.equation == "heat" else s1d.Equation.Euler
    scheme = s1d.Scheme.Swept if args.scheme == "swept" else s1d.Scheme.Classic
    n_total = n_per * world
    if world > 1:
        # One process per GPU: this rank owns shard `rank` of the ring; the
        # neighbours' boundary edges are read in place over NVLink.
        from paper_1811_08282_b200.dist import open_ring_shard
        cfg = s1d.LaunchConfig(equation=eq, scheme=scheme, grid_size=n_total, block_width=args.w, ranks=world,
                               steps=args.T)
        solver = open_ring_shard(cfg, rank, world, local)
        ring = ring_connect_record(rank, world, local, solver)
    else:
        cfg = s1d.LaunchConfig(equation=eq, scheme=scheme, grid_size=n_per, block_width=args.w, ranks=1,
                               steps=args.T, num_devices=1)
        solver = s1d.Solver(cfg)
        ring = {"nranks": 1, "devices": [local], "transport": "single shard (periodic ring of one)"}
    # warm-up
    for _ in range(args.warmup):
        solver.advance()
    barrier(world)
    loop_s, dom_s, dom_upd, dom_launch, launches = 0.0, 0.0, 0, 0, 0
    t0 = time.perf_counter()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            st, tm = solver.advance()
            loop_s += tm.loop_seconds
            dom_s += tm.dominant_seconds
            dom_upd += tm.dominant_point_updates
            dom_launch += tm.dominant_launches
            launches += st.kernel_launches
            dom_name = tm.dominant_kernel
    wall = time.perf_counter() - t0
    barrier(world)
    loop_s = allmax(world, loop_s)
    clocks = clk.summary()
    ms_per_step = 1e3 * loop_s / args.steps
    value = n_total * args.T * args.steps / loop_s / 1e6

    # e2e: same solve through the C ABI with pinned host buffers.
    e2e = None
    try:
        import torch
        hin = torch.empty(n_per, dtype=torch.float64, pin_memory=True)
        hout = torch.empty(n_per, dtype=torch.float64, pin_memory=True)
        s1d.initial_condition_range(cfg.initial_or_default(), n_total, cfg.spec(), solver.start, solver.count,
                                    cfg.phys.gamma, out=hin.numpy())
        solver.solve_ptr(hin.data_ptr(), n_per, hout.data_ptr(), n_per)  # warm
        e2e_times = []
        for _ in range(args.e2e_steps):
            t1 = time.perf_counter()
            solver.solve_ptr(hin.data_ptr(), n_per, hout.data_ptr(), n_per)
            e2e_times.append(time.perf_counter() - t1)
        e2e_t = allmax(world, sum(e2e_times))
        e2e = {"value": round(n_total * args.T * len(e2e_times) / e2e_t / 1e6, 3), "unit": UNIT,
               "h2d_bytes_per_step": 8 * n_per, "d2h_bytes_per_step": 8 * n_per,
               "ms_per_step": round(1e3 * e2e_t / len(e2e_times), 3)}
    except Exception as ex:  # pragma: no cover - reported, not hidden
        e2e = {"value": None, "unit": UNIT, "error": repr(ex)}

    # Roofline of the dominant kernel (the swept Diamond phases): FP64-pipe
    # bound. Algorithmic FP64 ops = 5 per point-update (DADD/DMUL; no FMA
    # contraction is allowed by bitwise parity) x point-updates per launch.
    fp64_peak = s1d.measure_fp64_peak(local)
    peaks = measured_peaks()
    roofline = None
    if dom_s > 0:
        # Roofline of the FP64 pipe, counted in instructions (DADD, DMUL and
        # DFMA each occupy it alike): the measured issue rate is the peak,
        # the minimum instructions per update under bitwise parity the work.
        ups = dom_upd / dom_s
        achieved = HEAT_FP64_INSTR_PER_UPDATE * ups
        roofline = {"bound": "fp64", "kernel": dom_name, "achieved": round(achieved / 1e12, 4),
                    "peak": round(fp64_peak / 1e12, 4), "unit": "T FP64-pipe instr/s",
                    "frac": round(achieved / fp64_peak, 4), "traffic": profile_traffic(args),
                    "peak_source": "measured in-run: s1d_measure_fp64_peak (DADD/DMUL issue-rate microkernel)",
                    "instr_per_update": HEAT_FP64_INSTR_PER_UPDATE,
                    "updates_per_launch": dom_upd // max(dom_launch, 1),
                    "algorithmic_dram_bytes_per_launch": 32 * n_per if dom_name == "swept_diamond" else None,
                    "traffic_note": "traffic = ncu dram read+write bytes per Diamond launch (profiles/traffic.json); "
                                    "algorithmic = the tiles' edge records in + out (4 doubles per point)",
                    "avg_launch_ms": round(1e3 * dom_s / max(dom_launch, 1), 4),
                    "flops_view": {"flops_per_update": HEAT_FLOPS_PER_UPDATE,
                                   "achieved_TFLOPs": round(HEAT_FLOPS_PER_UPDATE * ups / 1e12, 4),
                                   "fma_peak_TFLOPs": round(2 * fp64_peak / 1e12, 4),
                                   "frac": round(HEAT_FLOPS_PER_UPDATE * ups / (2 * fp64_peak), 4)},
                    "round1_basis": {"note": "5 ops per update against the DADD/DMUL issue rate (round 1's frac; "
                                             "no longer an upper bound once one op pair is fused)",
                                     "frac": round(HEAT_FLOPS_PER_UPDATE * ups / fp64_peak, 4)}}
        hbm = peaks.get("hbm_gbs")
        eq_gbs = CLASSIC_BYTES_PER_UPDATE * dom_upd / dom_s / 1e9
        roofline["hbm_equivalent"] = {"classic_bytes_per_update": CLASSIC_BYTES_PER_UPDATE,
                                      "achieved_GBps": round(eq_gbs, 1), "peak_GBps": hbm,
                                      "frac": round(eq_gbs / hbm, 3) if hbm else None,
                                      "note": "swept keeps levels on chip; >1 means it beats the classic "
                                              "scheme's HBM roofline"}

    # Classic comparison on the same grid (the metric is swept vs classic).
    classic = None
    if args.compare_classic and scheme == s1d.Scheme.Swept and world == 1:
        ccfg = s1d.LaunchConfig(equation=eq, scheme=s1d.Scheme.Classic, grid_size=n_per, block_width=args.w,
                                ranks=1, steps=args.classic_T, num_devices=1)
        with s1d.Solver(ccfg) as cs:
            cs.advance()
            ct = min(cs.advance()[1].loop_seconds for _ in range(2))
        crate = n_per * args.classic_T / ct / 1e6
        classic = {"value": round(crate, 3), "unit": UNIT, "steps_per_run": args.classic_T,
                   "us_per_timestep": round(1e6 * ct / args.classic_T, 3),
                   "hbm_GBps": round(CLASSIC_BYTES_PER_UPDATE * n_per * args.classic_T / ct / 1e9, 1),
                   "swept_speedup": round(value / world / crate, 3)}

    # Secondary configuration (BASELINE configs[2]): Euler Sod, both methods,
    # swept vs classic on this GPU. Point-update = one point x one time step.
    euler = None
    if args.euler and world == 1:
        euler = {"grid_size": 1 << args.euler_log2n, "block_width": args.euler_w, "steps_per_run": args.euler_T,
                 "unit": "Mpt-steps/s"}
        for meth in ("lengthening", "flattening"):
            for sch in ("swept", "classic"):
                ecfg = s1d.LaunchConfig(equation=s1d.Equation.Euler,
                                        method=s1d.Method.Lengthening if meth == "lengthening"
                                        else s1d.Method.Flattening,
                                        scheme=s1d.Scheme.Swept if sch == "swept" else s1d.Scheme.Classic,
                                        grid_size=1 << args.euler_log2n, block_width=args.euler_w, ranks=1,
                                        steps=args.euler_T if sch == "swept" else max(args.euler_T // 8, 16),
                                        num_devices=1)
                with s1d.Solver(ecfg) as es:
                    es.advance()
                    best = min(es.advance()[1].loop_seconds for _ in range(2))
                euler[f"{meth}_{sch}"] = round(ecfg.grid_size * ecfg.steps / best / 1e6, 2)
            euler[f"{meth}_swept_speedup"] = round(euler[f"{meth}_swept"] / euler[f"{meth}_classic"], 3)
        euler["roofline"] = euler_pipe_profile()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = host_cores()
            n_s, t_s, _ = reference_sample_size(args, 1)
            rate, ranks, secs = cpu_reference_sample(args.equation, args.scheme, args.w, n_s, t_s, threads)
            cpu = {"value": round(rate / 1e6, 3), "unit": UNIT, "cores": ranks, "kind": "reference",
                   "host_cores": threads, "cpu_model": cpu_model(),
                   "sample": f"sweep1d::run({args.scheme}, WallClock) n=2^{n_s.bit_length() - 1} "
                             f"w={args.w} T={t_s}, {ranks} rank threads, {secs:.1f} s"}
        except Exception as ex:
            cpu = {"value": None, "unit": UNIT, "error": repr(ex)}

    solver.close()
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: the reference's heat-sine initial condition (partition.cpp:54-73)",
            "config": {"workload": workload_name(args), "equation": args.equation, "scheme": args.scheme,
                       "grid_size": n_total, "grid_per_gpu": n_per, "block_width": args.w,
                       "steps_per_run": args.T, "parallelism": f"shards{world}",
                       "l2": "inputs larger than L2 (1 GiB state per GPU vs 126 MB L2)"},
            "us_per_timestep": round(1e6 * loop_s / args.steps / args.T, 3),
            "clocks": clocks, "e2e": e2e, "gpu_launches": launches, "roofline": roofline, "ring": ring,
            "classic_same_grid": classic, "euler_sod": euler, "cpu_baseline": cpu,
            "wall_seconds_timed_region": round(wall, 3),
        }
        print(json.dumps(line), flush=True)
    return 0


def profile_traffic(args):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    capture (profiles/), when one exists for this configuration."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            table = json.load(fh)
        return table.get(f"{args.equation}-{args.scheme}-w{args.w}")
    except Exception:
        return None


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--equation", choices=["heat"], default="heat")
    ap.add_argument("--scheme", choices=["swept", "classic"], default="swept")
    ap.add_argument("--log2n", type=int, default=27)
    ap.add_argument("--w", type=int, default=1024, help="block width (the sweep's best at n = 2^27, T = 6144)")
    ap.add_argument("--T", type=int, default=6144)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--classic-T", type=int, default=256)
    ap.add_argument("--no-compare-classic", dest="compare_classic", action="store_false")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-euler", dest="euler", action="store_false", help="skip the Euler (configs[2]) lines")
    ap.add_argument("--euler-log2n", type=int, default=22)
    ap.add_argument("--euler-w", type=int, default=512)
    ap.add_argument("--euler-T", type=int, default=1024)
    ap.add_argument("--ref-n", type=int, default=0, help="CPU reference sample grid size (default: 2^log2n)")
    ap.add_argument("--ref-steps", type=int, default=0, help="CPU reference sample time steps (default: w/2)")
    ap.add_argument("--ref-budget-s", type=float, default=420.0,
                    help="upper bound on the reference arm's timed CPU work (n is halved to fit)")
    args = ap.parse_args(argv)
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(sys.argv[1:] if argv is None else argv, args.gpus)
    rank, world = dist_init()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started {world} processes")
    if args.impl == "reference":
        return run_reference_arm(args, rank, world)
    return run_b200(args, rank, world)


if __name__ == "__main__":
    sys.exit(main())

"""alpha-beta model calibrated on NVLink vs measured multi-GPU runs.

    python -m torch.distributed.run --nproc-per-node G --master-addr 127.0.0.1 \
        tools/alpha_beta.py [--out gpurun_out/alpha_beta.json]

1. rank 0 calibrates alpha (one-way device flag hand-off over NVLink, the
   swept round's synchronisation) and beta (s/byte of a peer copy) between
   devices 0 and 1 (s1d_calibrate_transport);
2. for each workload, rank 0 measures the per-point-substep cost on one GPU
   (same points per GPU, ranks = 1) -> compute_cost;
3. all ranks run the workload one process per GPU (the production path) and
   report the device time per step (max over ranks);
4. the reference's virtual clock (s1d_virtual_time) with the calibrated
   (alpha, beta, compute_cost) predicts the G-GPU time per step. The residual
   per round, (measured - predicted) / rounds, is the engine's per-round
   overhead beyond the hardware hand-off (kernel launches on the round's
   critical path), reported as alpha_eff.
"""
import argparse
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1811_08282_b200 as s1d  # noqa: E402
from paper_1811_08282_b200.dist import open_ring_shard  # noqa: E402

H, E = s1d.Equation.Heat, s1d.Equation.Euler
L, F = s1d.Method.Lengthening, s1d.Method.Flattening
SW, CL = s1d.Scheme.Swept, s1d.Scheme.Classic
# (name, equation, method, scheme, points per GPU, w, T)
WORKLOADS = [
    ("heat swept 2^27/GPU", H, L, SW, 1 << 27, 1024, 6144),
    ("heat classic 2^27/GPU", H, L, CL, 1 << 27, 1024, 512),
    ("heat swept 2^20/GPU", H, L, SW, 1 << 20, 1024, 6144),
    ("heat classic 2^20/GPU", H, L, CL, 1 << 20, 1024, 2048),
    ("euler-len swept 2^16/GPU", E, L, SW, 1 << 16, 512, 2048),
    ("euler-len classic 2^16/GPU", E, L, CL, 1 << 16, 512, 512),
    ("euler-flat swept 2^16/GPU", E, F, SW, 1 << 16, 512, 2048),
    ("euler-flat classic 2^16/GPU", E, F, CL, 1 << 16, 512, 512),
]


def best_time(solver, reps=3):
    solver.advance()
    return min(solver.advance()[1].loop_seconds for _ in range(reps))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/alpha_beta.json")
    args = ap.parse_args()
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = int(os.environ.get("LOCAL_RANK", rank))
    tp = torch.zeros(2, dtype=torch.float64)
    if rank == 0:
        t = s1d.calibrate_transport(0, 1)
        tp[:] = torch.tensor([t.alpha, t.beta])
    dist.broadcast(tp, 0)
    alpha, beta = float(tp[0]), float(tp[1])
    rows = []
    for name, eq, me, sc, per, w, T in WORKLOADS:
        cfg = s1d.LaunchConfig(equation=eq, method=me, scheme=sc, grid_size=per * world, block_width=w, ranks=world,
                               steps=T, mode=s1d.Mode.WallClock)
        S = cfg.spec().substeps_per_step
        cc = torch.zeros(1, dtype=torch.float64)
        if rank == 0:
            one = dataclasses.replace(cfg, grid_size=per, ranks=1, num_devices=1)
            with s1d.Solver(one) as sv:
                cc[0] = best_time(sv) / (per * T * S)
        dist.broadcast(cc, 0)
        with open_ring_shard(cfg, rank, world, dev) as sh:
            t = torch.tensor([best_time(sh)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            model = dataclasses.replace(cfg, mode=s1d.Mode.VirtualTime,
                                        transport=s1d.TransportParams(alpha, beta, float(cc[0])))
            v, comm = s1d.virtual_time(model)
            m = s1d.cycle_advance(w, cfg.spec().stencil_half_width)
            rounds = T * S if sc == CL else (T * S) // m + (T * S) % m
            meas, pred = float(t[0]) / T, v / T
            row = dict(workload=name, gpus=world, T=T, compute_cost_s=float(cc[0]), rounds=rounds,
                       measured_us_per_step=meas * 1e6, predicted_us_per_step=pred * 1e6,
                       model_comm_us_per_step=comm / T * 1e6, rel_error=(pred - meas) / meas,
                       alpha_eff_s=(meas - pred) * T / rounds + alpha)
            rows.append(row)
            print(f"{name:30s} G={world} measured {row['measured_us_per_step']:10.2f} us/step  "
                  f"model {row['predicted_us_per_step']:10.2f} (comm {row['model_comm_us_per_step']:7.3f})  "
                  f"err {100 * row['rel_error']:+6.1f}%  alpha_eff {row['alpha_eff_s'] * 1e6:7.2f} us", flush=True)
    if rank == 0:
        out = dict(gpus=world, alpha_s=alpha, beta_s_per_byte=beta, peer_copy_GBps=1e-9 / beta, rows=rows)
        print(f"calibrated: alpha = {alpha * 1e6:.3f} us (one-way NVLink flag hand-off), "
              f"beta = {beta * 1e12:.4f} ps/B ({1e-9 / beta:.1f} GB/s peer copy)")
        os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
        json.dump(out, open(args.out, "w"), indent=1)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Multi-process parity check (torchrun, one process per GPU):
    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/mp_check.py
Each rank runs its shard; rank 0 gathers the slices and compares the global
state with the CPU oracle, bit for bit. Exit code 0 = all cases pass."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1811_08282_b200 as s1d  # noqa: E402
from paper_1811_08282_b200.dist import open_ring_shard  # noqa: E402

CASES = [
    # equation, method, scheme, n, w, wf, steps
    ("heat", "lengthening", "swept", 1 << 14, 64, 0, 1000),
    ("heat", "lengthening", "classic", 1 << 14, 64, 0, 300),
    ("heat", "lengthening", "swept", 1 << 12, 32, 0, 77),     # unaligned: classic pad across shards
    ("heat", "lengthening", "swept", 1 << 14, 1024, 0, 2048),
    ("heat", "lengthening", "swept", 1 << 12, 64, 3, 200),    # fat rank 0
    ("euler", "lengthening", "swept", 1 << 12, 64, 0, 250),
    ("euler", "lengthening", "classic", 1 << 12, 64, 0, 40),
    ("euler", "flattening", "swept", 1 << 12, 128, 0, 111),
    ("euler", "flattening", "classic", 1 << 12, 64, 0, 30),
    # 96 blocks: partitions for 2, 3, 4, 6 and 8 ranks
    ("heat", "lengthening", "swept", 96 * 64, 64, 0, 333),
    ("heat", "lengthening", "classic", 96 * 64, 64, 0, 50),
    ("euler", "lengthening", "swept", 96 * 64, 64, 0, 77),
    ("euler", "flattening", "swept", 96 * 64, 64, 0, 61),
]

WAVE_CASES = [
    # equation, method, n, w, steps, S1D_WAVE shape (96 tiles: >= 12 per rank up to 8 ranks)
    ("heat", "lengthening", 96 * 64, 64, 32 * 9, "16,3,3"),
    ("heat", "lengthening", 96 * 256, 256, 128 * 9, None),
    ("heat", "lengthening", 96 * 64, 64, 32 * 10, "5,1,2"),
    ("euler", "lengthening", 96 * 64, 64, 72, "16,2,2"),
    ("euler", "flattening", 96 * 64, 64, 80, "7,1,1"),
]


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    failures = 0
    for eq, me, sc, n, w, wf, T in CASES:
        if wf and world == 1:
            wf = 0
        cfg = s1d.LaunchConfig(equation=s1d.Equation.Heat if eq == "heat" else s1d.Equation.Euler,
                               method=s1d.Method.Lengthening if me == "lengthening" else s1d.Method.Flattening,
                               scheme=s1d.Scheme.Swept if sc == "swept" else s1d.Scheme.Classic, grid_size=n,
                               block_width=w, ranks=world, work_factor=wf, steps=T)
        try:
            s1d.make_partition(cfg)
        except s1d.InvalidConfig:  # e.g. WF shares that do not divide the blocks at this world size
            if rank == 0:
                print(f"skip {eq} {me} {sc} n={n} w={w} wf={wf}: no partition for {world} ranks", flush=True)
            continue
        with open_ring_shard(cfg) as shard:
            out, st, tm = shard.solve()
            out2, _, _ = shard.solve()  # repeated runs stay in lockstep
            same = np.array_equal(out.view(np.uint64), out2.view(np.uint64))
            parts = [None] * world
            dist.all_gather_object(parts, (shard.start, out, same, st.exchange_rounds))
        if rank == 0:
            vpp = 1 if eq == "heat" else 3
            glob = np.empty(n * vpp)
            for start, arr, _, _ in parts:
                glob[start * vpp: start * vpp + arr.size] = arr
            from oracle import oracle as O
            want = O.port_run_serial(eq, me, n=n, steps=T)
            ok = np.array_equal(glob.view(np.uint64), want.view(np.uint64)) and all(p[2] for p in parts)
            failures += not ok
            print(f"{'ok ' if ok else 'BAD'} {eq}/{me}/{sc} n={n} w={w} wf={wf} T={T} ranks={world} "
                  f"rounds={parts[0][3]} loop={tm.loop_seconds * 1e3:.2f} ms", flush=True)
    # wavefront solve across processes (engine.cu wavefront_phases: end chunks
    # behind the neighbours' round flags, per-phase signals); S1D_WAVE forces
    # a shape, None = the default (heat m <= 128)
    for eq, me, n, w, T, shape in WAVE_CASES:
        if shape:
            os.environ["S1D_WAVE"] = shape
        else:
            os.environ.pop("S1D_WAVE", None)
        cfg = s1d.LaunchConfig(equation=s1d.Equation.Heat if eq == "heat" else s1d.Equation.Euler,
                               method=s1d.Method.Lengthening if me == "lengthening" else s1d.Method.Flattening,
                               scheme=s1d.Scheme.Swept, grid_size=n, block_width=w, ranks=world, steps=T)
        with open_ring_shard(cfg) as shard:
            out, _, tm = shard.solve()
            out2, _, _ = shard.solve()
            same = np.array_equal(out.view(np.uint64), out2.view(np.uint64))
            parts = [None] * world
            dist.all_gather_object(parts, (shard.start, out, same))
        if rank == 0:
            vpp = 1 if eq == "heat" else 3
            glob = np.empty(n * vpp)
            for start, arr, _ in parts:
                glob[start * vpp: start * vpp + arr.size] = arr
            from oracle import oracle as O
            want = O.port_run_serial(eq, me, n=n, steps=T)
            ok = np.array_equal(glob.view(np.uint64), want.view(np.uint64)) and all(p[2] for p in parts)
            failures += not ok
            print(f"{'ok ' if ok else 'BAD'} wavefront {eq}/{me} n={n} w={w} T={T} shape={shape or 'default'} "
                  f"ranks={world} dominant={tm.dominant_launches}", flush=True)
    os.environ.pop("S1D_WAVE", None)
    # heat fast form's guard across processes (heat.cu heat_step): a spike
    # >= 2^1022 near rank 0's right seam flags rank 0's Up; the flag spreads
    # to the neighbours' launches through the IPC-shared flag words, the gated
    # exact builds recompute, and the result is the oracle's, bit for bit
    # (T = 700: classic pad, Up/Down pipeline; T = 1152: 9 cycles, wavefront)
    for T in (700, 1152):
        n, w = 96 * 256, 256
        cfg = s1d.LaunchConfig(equation=s1d.Equation.Heat, scheme=s1d.Scheme.Swept, grid_size=n, block_width=w,
                               ranks=world, steps=T)
        x = np.arange(n)
        u0 = np.sin(2 * np.pi * x / n) + 0.3 * np.cos(0.37 * x)
        u0[n // world - 5] = 1.6 * 2.0 ** 1022
        with open_ring_shard(cfg) as shard:
            out, _, _ = shard.solve(u0[shard.start:shard.start + shard.count])
            parts = [None] * world
            dist.all_gather_object(parts, (shard.start, out))
        if rank == 0:
            from oracle import oracle as O
            glob = np.empty(n)
            for start, arr in parts:
                glob[start:start + arr.size] = arr
            want = O.port_run_state("heat", "lengthening", u0, T, 0.0)
            ok = np.array_equal(glob.view(np.uint64), want.view(np.uint64))
            failures += not ok
            print(f"{'ok ' if ok else 'BAD'} heat fast-form guard, spike >= 2^1022, n={n} w={w} T={T} ranks={world}",
                  flush=True)
    dist.barrier()
    code = [failures]
    dist.broadcast_object_list(code, src=0)
    dist.destroy_process_group()
    sys.exit(1 if code[0] else 0)


if __name__ == "__main__":
    main()

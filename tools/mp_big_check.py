"""One-process-per-rank parity at bench size (torchrun; ranks may share a GPU):
    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/mp_big_check.py
Each rank solves its shard (heat 2^27 points per rank, w = 1024, the bench's
configuration; Euler Sod 2^16 points per rank, both methods) and publishes a
SHA-256 of its slice; rank 0 then solves the whole grid as one shard and
compares slice by slice (rank invariance, R/tests/test_decomp.cpp:81-98).
Exit code 0 = all cases pass."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch.distributed as dist  # noqa: E402

import paper_1811_08282_b200 as s1d  # noqa: E402
from paper_1811_08282_b200.dist import open_ring_shard  # noqa: E402

CASES = [
    # equation, method, log2 points per rank, w, steps
    ("heat", "lengthening", 27, 1024, 2048),
    ("heat", "lengthening", 27, 1024, 700),  # unaligned: classic pad across the seams
    ("euler", "lengthening", 16, 512, 1024),
    ("euler", "flattening", 16, 512, 1024),
]


def digest(a):
    return hashlib.sha256(a.tobytes()).hexdigest()


def config(eq, me, n, w, T, ranks):
    return s1d.LaunchConfig(equation=s1d.Equation.Heat if eq == "heat" else s1d.Equation.Euler,
                            method=s1d.Method.Lengthening if me == "lengthening" else s1d.Method.Flattening,
                            scheme=s1d.Scheme.Swept, grid_size=n, block_width=w, ranks=ranks, steps=T,
                            mode=s1d.Mode.WallClock)


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    failures = 0
    for eq, me, lg, w, T in CASES:
        n = world << lg
        with open_ring_shard(config(eq, me, n, w, T, world)) as shard:
            out, st, tm = shard.solve()
            parts = [None] * world
            dist.all_gather_object(parts, (shard.start, shard.count, digest(out), tm.loop_seconds))
        dist.barrier()
        if rank == 0:
            cfg = config(eq, me, n, w, T, 1)
            cfg.num_devices = 1
            ref = s1d.run(cfg).state
            vpp = 1 if eq == "heat" else 3
            ok = all(digest(ref[start * vpp:(start + count) * vpp]) == h for start, count, h, _ in parts)
            failures += not ok
            print(f"{'ok ' if ok else 'BAD'} {eq}/{me} n={n} ({world} x 2^{lg}) w={w} T={T} "
                  f"loop={max(p[3] for p in parts) * 1e3:.1f} ms", flush=True)
        dist.barrier()
    code = [failures]
    dist.broadcast_object_list(code, src=0)
    dist.destroy_process_group()
    sys.exit(1 if code[0] else 0)


if __name__ == "__main__":
    main()

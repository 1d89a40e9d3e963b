"""Config 5 probe (torchrun): Euler Sod, 2^16 points per GPU, long T, swept vs
classic across block widths, one process per GPU. Prints one line per config
(rank 0): device time per step (max over ranks) and point-steps/s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1811_08282_b200 as s1d  # noqa: E402
from paper_1811_08282_b200.dist import open_ring_shard  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    per = int(os.environ.get("PER", 1 << 16))
    T = int(os.environ.get("T", 2048))
    for method in ("lengthening", "flattening"):
        for scheme, ws in (("classic", [64]), ("swept", [64, 128, 256, 512, 1024])):
            for w in ws:
                cfg = s1d.LaunchConfig(equation=s1d.Equation.Euler,
                                       method=s1d.Method.Lengthening if method == "lengthening"
                                       else s1d.Method.Flattening,
                                       scheme=s1d.Scheme.Swept if scheme == "swept" else s1d.Scheme.Classic,
                                       grid_size=per * world, block_width=w, ranks=world,
                                       steps=T if scheme == "swept" else T // 4)
                with open_ring_shard(cfg) as sh:
                    sh.advance()
                    best = min(sh.advance()[1].loop_seconds for _ in range(3))
                t = torch.tensor([best], dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                if rank == 0:
                    sec = t.item()
                    print(f"{world} GPUs euler {method} {scheme} w={w} n={per}x{world}: {1e6 * sec / cfg.steps:9.2f} "
                          f"us/step {cfg.grid_size * cfg.steps / sec / 1e9:7.2f} Gpt-steps/s", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

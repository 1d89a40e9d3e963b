"""GPU multi-device parity (single-device cases run anywhere; the rest need 2 GPUs):
  * single process, shards on several devices (ranks = G, num_devices = G);
  * one process per GPU (torchrun + CUDA IPC + device flags): tools/mp_check.py.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1811_08282_b200 as s1d
from oracle import oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ngpu():
    return s1d.device_count()


need2 = pytest.mark.skipif(ngpu() < 2, reason="needs >= 2 GPUs")


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


@need2
@pytest.mark.parametrize("eq,method", [("heat", "lengthening"), ("euler", "lengthening"), ("euler", "flattening")])
@pytest.mark.parametrize("scheme", [s1d.Scheme.Swept, s1d.Scheme.Classic], ids=s1d.to_string)
@pytest.mark.parametrize("ranks,wf", [(2, 0), (3, 0), (4, 2)])
def test_single_process_multi_device(gpu, eq, method, scheme, ranks, wf):
    n, w, T = 60 * 64, 64, 137  # 60 blocks: divisible by 2, 3 and 5 shares
    cfg = s1d.LaunchConfig(equation=s1d.Equation.Heat if eq == "heat" else s1d.Equation.Euler,
                           method=s1d.Method.Lengthening if method == "lengthening" else s1d.Method.Flattening,
                           scheme=scheme, grid_size=n, block_width=w, ranks=ranks, work_factor=wf, steps=T,
                           num_devices=min(ngpu(), ranks))
    got = s1d.run(cfg).state
    assert np.array_equal(bits(got), bits(O.port_run_serial(eq, method, n=n, steps=T)))


def _torchrun_mp_check(nproc, port):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "tools", "mp_check.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0
    assert "BAD" not in r.stdout
    return r.stdout.count("ok ")


@need2
def test_multi_process_torchrun(gpu):
    # one process per GPU, the bench contract's launch mode
    assert _torchrun_mp_check(2, 29517) >= 19


def test_multi_process_ranks_share_gpus(gpu):
    # more ranks than GPUs (ranks wrap onto devices): the CUDA IPC + device
    # flag ring with 4 processes, runnable on a single-GPU box
    assert _torchrun_mp_check(4, 29518) >= 18

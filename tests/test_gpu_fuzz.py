"""GPU parity over seeded random configurations: equation / method / scheme,
block width (short-tile, P = 2/4/8/16 paths), shard count and work factor
(shards share the visible devices), unaligned step counts (classic pad) —
bitwise against the CPU oracle. Invalid draws (the reference's validation
rejects them) are skipped, so every case that runs is a configuration the
reference accepts."""
import numpy as np
import pytest

import paper_1811_08282_b200 as s1d
from oracle import oracle as O

pytestmark = pytest.mark.gpu

WIDTHS = [4, 6, 8, 10, 12, 16, 20, 24, 32, 40, 48, 64, 96, 128, 192, 256, 320, 512]


def draw(seed):
    r = np.random.default_rng(seed)
    eq = "heat" if r.random() < 0.5 else "euler"
    method = "lengthening" if r.random() < 0.5 else "flattening"
    scheme = s1d.Scheme.Swept if r.random() < 0.75 else s1d.Scheme.Classic
    w = int(r.choice(WIDTHS))
    ranks = int(r.integers(1, 5))
    wf = int(r.choice([0, 0, 1, 2]))
    shares = ranks - 1 + wf if wf else ranks  # make_partition: rank 0 takes WF shares
    blocks = shares * int(r.integers(1, 5))
    n = blocks * w
    steps = int(r.integers(1, 120 if eq == "euler" else 400))
    return eq, method, scheme, n, w, ranks, wf, steps


@pytest.mark.parametrize("seed", range(150))
def test_random_configuration_matches_oracle(gpu, seed):
    eq, method, scheme, n, w, ranks, wf, steps = draw(1000 + seed)
    cfg = s1d.LaunchConfig(equation=s1d.Equation.Heat if eq == "heat" else s1d.Equation.Euler,
                           method=s1d.Method.Lengthening if method == "lengthening" else s1d.Method.Flattening,
                           scheme=scheme, grid_size=n, block_width=w, ranks=ranks, work_factor=wf, steps=steps,
                           mode=s1d.Mode.WallClock, num_devices=min(ranks, max(1, s1d.device_count())))
    try:
        cfg.validate(True)
        s1d.make_partition(cfg)
    except (s1d.InvalidConfig, s1d.InvalidWidth):
        pytest.skip("configuration rejected by the reference's validation")
    try:
        got = s1d.run(cfg).state
    except s1d.InvalidWidth:
        pytest.skip("width has no tile decomposition")
    want = O.port_run_serial(eq, method, n=n, steps=steps)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (eq, method, scheme, n, w, ranks, wf, steps)

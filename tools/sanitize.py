"""Small runs of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck). Usage: compute-sanitizer --tool racecheck python tools/sanitize.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1811_08282_b200 as s1d  # noqa: E402
from oracle import oracle as O  # noqa: E402

CASES = [  # eq, method, scheme, n, w, steps
    ("heat", "lengthening", "swept", 64 * 32, 32, 50),      # short tiles (staged exports), pad
    ("heat", "lengthening", "swept", 8 * 128, 128, 100),    # P = 16, streamed ring
    ("heat", "lengthening", "swept", 4 * 1024, 1024, 1100), # wide tiles
    ("heat", "lengthening", "swept", 6 * 6, 6, 20),         # P = 2
    ("heat", "lengthening", "classic", 2048, 64, 20),
    ("euler", "lengthening", "swept", 16 * 64, 64, 20),
    ("euler", "flattening", "swept", 8 * 128, 128, 40),
    ("euler", "lengthening", "classic", 1024, 64, 5),
    ("euler", "flattening", "classic", 1024, 64, 5),
]
bad = 0
for eq, me, sc, n, w, T in CASES:
    cfg = s1d.LaunchConfig(equation=s1d.Equation.Heat if eq == "heat" else s1d.Equation.Euler,
                           method=s1d.Method.Lengthening if me == "lengthening" else s1d.Method.Flattening,
                           scheme=s1d.Scheme.Swept if sc == "swept" else s1d.Scheme.Classic, grid_size=n,
                           block_width=w, ranks=2 if n % (2 * w) == 0 else 1, steps=T, mode=s1d.Mode.WallClock,
                           num_devices=1)
    ok = np.array_equal(s1d.run(cfg).state.view(np.uint64), O.port_run_serial(eq, me, n=n, steps=T).view(np.uint64))
    bad += not ok
    print(("ok " if ok else "BAD"), eq, me, sc, n, w, T, "ranks", cfg.ranks, flush=True)
sys.exit(1 if bad else 0)

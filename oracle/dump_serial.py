"""TEST INFRASTRUCTURE ONLY — write the reference's serial oracle state for a
configuration as a raw little-endian float64 dump, the `--against` input of
`s1d verify` (SPEC.md bench-cli: "verify (swept vs classic vs serial
oracle)").

    python oracle/dump_serial.py --out F.bin [--port] key=value ...

Keys are the CLI's (equation method n w steps initial fourier gamma cfl).
By default the dump comes from the unmodified reference compiled from source
(oracle/_ref: sweep1d::run_serial, inc/engine.hpp:32); --port uses this
repo's C restatement (oracle/s1d_oracle.c) where oracle/_ref is absent.
"""
from __future__ import annotations

import argparse
import os
import sys

sys.path[0] = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))  # not oracle/ itself

from oracle import oracle as O  # noqa: E402


def parse_kv(items):
    cfg = {}
    for it in items:
        k, _, v = it.partition("=")
        k = {"grid_size": "n", "block_width": "w"}.get(k, k)
        if k == "n" and v.startswith("2^"):
            v = str(1 << int(v[2:]))
        cfg[k] = v
    return cfg


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--out", required=True)
    ap.add_argument("--port", action="store_true", help="use the C restatement instead of the compiled reference")
    ap.add_argument("kv", nargs="*")
    a = ap.parse_args(argv)
    kv = parse_kv(a.kv)
    eq = kv.get("equation", "heat")
    me = kv.get("method", "lengthening")
    n = int(kv.get("n", 1024))
    steps = int(kv.get("steps", 50))
    fo, gamma, cfl = float(kv.get("fourier", 0.4)), float(kv.get("gamma", 1.4)), float(kv.get("cfl", 0.4))
    initial = kv.get("initial", "")
    if a.port or not O.ref_available():
        state = O.port_run_serial(eq, me, n=n, steps=steps, fourier=fo, gamma=gamma, cfl=cfl, initial=initial)
        src = "port"
    else:
        cfg = O.RefConfig(equation=eq, method=me, grid_size=n, block_width=int(kv.get("w", 32)), ranks=2,
                          steps=steps, initial=initial, fourier=fo, gamma=gamma, cfl=cfl)
        state = O.ref_run_serial(cfg)
        src = "reference"
    state.astype("<f8").tofile(a.out)
    print(f"wrote {state.size} doubles ({src} run_serial, {eq}/{me} n={n} T={steps}) to {a.out}")


if __name__ == "__main__":
    main()

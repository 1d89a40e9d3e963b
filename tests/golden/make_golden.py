"""Generate tests/golden/golden.json from the reference compiled from source
(oracle/_ref/libsweep1d_ref.so). Run in the dev container, where
/root/reference is mounted:  python tests/golden/make_golden.py

Contents (every value produced by the UNMODIFIED reference code):
  * fingerprints: FNV-1a-64 of run_serial output for the SURVEY.md §8c
    configurations (+ a few more), with sample values;
  * decomp: full run_serial states for the nine test_decomp.cpp:108-118 cases
    and the classic rank-invariance case (:84), small enough to store;
  * kernels: per-point known answers (heat_step, minmod, pressure ratio,
    interface flux, the Sod predictor of test_kernels.cpp:184-197);
  * ic / dt_dx / partition / schedules known answers.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402


def floats(a):
    return [float(x) for x in np.asarray(a).ravel()]


def main():
    g = {"generator": "tests/golden/make_golden.py via oracle/_ref/libsweep1d_ref.so (reference compiled from "
                      "/root/reference/proj/core/src)"}
    fps = []
    for eq, me, n, T in [("heat", "lengthening", 1 << 14, 64), ("heat", "lengthening", 1 << 14, 1000),
                         ("heat", "lengthening", 1 << 14, 6144), ("euler", "lengthening", 1 << 14, 64),
                         ("euler", "flattening", 1 << 14, 64), ("euler", "lengthening", 1 << 14, 250),
                         ("euler", "flattening", 1 << 12, 300), ("heat", "lengthening", 1 << 10, 3333),
                         ("euler", "lengthening", 1 << 10, 2000)]:
        st = O.ref_run_serial(O.RefConfig(equation=eq, method=me, grid_size=n, block_width=64, steps=T))
        fps.append({"equation": eq, "method": me, "n": n, "steps": T, "fnv1a64": O.fnv1a64(st),
                    "sample": {str(i): float(st[i]) for i in (1, 7, len(st) // 4, len(st) // 2 + 1)}})
    g["fingerprints"] = fps

    cases = [("heat", "lengthening", 64, 4, 2, 0, 16), ("heat", "lengthening", 32, 8, 2, 0, 4),
             ("heat", "lengthening", 128, 8, 3, 2, 25), ("heat", "lengthening", 64, 8, 2, 0, 21),
             ("euler", "lengthening", 96, 8, 3, 0, 10), ("euler", "lengthening", 64, 16, 2, 0, 7),
             ("euler", "flattening", 96, 8, 2, 0, 10), ("euler", "flattening", 128, 8, 4, 0, 3),
             ("euler", "flattening", 128, 16, 2, 0, 5), ("euler", "lengthening", 192, 8, 3, 4, 8),
             ("heat", "lengthening", 128, 32, 2, 0, 50)]
    dec = []
    for eq, me, n, w, r, wf, T in cases:
        cfg = O.RefConfig(equation=eq, method=me, scheme="swept", grid_size=n, block_width=w, ranks=r,
                          work_factor=wf, steps=T)
        serial = O.ref_run_serial(cfg)
        swept = O.ref_run(cfg, keep_log=True)
        cfg.scheme = "classic"
        classic = O.ref_run(cfg)
        assert np.array_equal(swept.state.view(np.uint64), serial.view(np.uint64))
        assert np.array_equal(classic.state.view(np.uint64), serial.view(np.uint64))
        dec.append({"equation": eq, "method": me, "n": n, "w": w, "ranks": r, "wf": wf, "steps": T,
                    "state": floats(serial), "fnv1a64": O.fnv1a64(serial),
                    "swept_rounds": swept.exchange_rounds, "swept_messages": swept.messages_sent,
                    "swept_bytes": swept.bytes_sent, "classic_rounds": classic.exchange_rounds,
                    "classic_messages": classic.messages_sent, "classic_bytes": classic.bytes_sent})
    g["decomp"] = dec

    lib = O.ref()
    k = {}
    k["heat_step"] = [[l, c, r, fo, lib.ref_heat_step(l, c, r, fo)] for l, c, r, fo in
                      [(1.0, 1.0, 1.0, 0.25), (0.0, 1.0, 0.0, 0.25), (1.0, 0.0, 0.0, 0.5), (0.37, -1.25, 2.6251, 0.4),
                       (1e-300, 3e-300, -2e-300, 0.4), (0.1, 0.2, 0.3, 0.5)]]
    vals = [-2.5, -1.0, -0.25, 0.0, -0.0, 0.75, 1.5, 3.0, float("inf"), float("-inf")]
    k["minmod"] = [[a, b, lib.ref_minmod(a, b)] for a in vals for b in vals]
    k["pressure_ratio"] = [[a, b, c, lib.ref_pressure_ratio_value(a, b, c)] for a, b, c in
                           [(1.0, 2.0, 4.0), (4.0, 2.0, 1.0), (1.0, 1.0, 1.0), (0.3, 0.7, 0.7000000000000001),
                            (1.0, 2.0, 2.0 + 1e-15), (2.0, 1.0, 3.0), (1.0, 1.0, 2.0)]]
    rng = np.random.default_rng(7)
    iflux = []
    for _ in range(64):
        ql = np.array([rng.uniform(0.1, 2), rng.uniform(-0.5, 0.5), 0.0])
        qr = np.array([rng.uniform(0.1, 2), rng.uniform(-0.5, 0.5), 0.0])
        ql[2] = rng.uniform(0.5, 3) / 0.4 + 0.5 * ql[1] ** 2 / ql[0]
        qr[2] = rng.uniform(0.5, 3) / 0.4 + 0.5 * qr[1] ** 2 / qr[0]
        prl, prr = rng.choice([rng.uniform(-2, 2), float("nan"), 0.0, -0.0]), rng.choice(
            [rng.uniform(-2, 2), float("nan"), 0.0, -0.0])
        out = np.empty(3)
        e = O._err()
        st = lib.ref_interface_flux(O._ptr(ql), O._ptr(qr), prl, prr, 1.4, O._ptr(out), e, 512)
        iflux.append({"ql": floats(ql), "qr": floats(qr), "pr_l": prl, "pr_r": prr, "status": st,
                      "flux": floats(out) if st == 0 else None})
    k["interface_flux"] = iflux
    # Sod predictor (test_kernels.cpp:184-197)
    def rec(rho, u, p):
        q = [rho, rho * u, p / 0.4 + 0.5 * rho * u * u]
        return q + q + [0.0]
    cells = np.array([rec(1, 0, 1), rec(1, 0, 1), rec(1, 0, 1), rec(0.125, 0, 0.1), rec(0.125, 0, 0.1)]).ravel()
    dt_dx = 0.4 / np.sqrt(1.4)
    for i in (1, 2, 3):
        O.ref_model_apply(1, cells, i, 1, gamma=1.4, dt_dx=dt_dx)
    O.ref_model_apply(1, cells, 2, 2, gamma=1.4, dt_dx=dt_dx)
    k["sod_predictor"] = {"q1": floats(cells[7 * 2 + 3: 7 * 2 + 6]),
                          "expect_1e-14": [0.91481618952839827, 0.076063882925566498, 2.2809559159301673]}
    g["kernels"] = k

    g["ic"] = {"heat-sine-4": floats(O.ref_initial_condition("heat-sine", 4)),
               "heat-sine-12": floats(O.ref_initial_condition("heat-sine", 12)),
               "sod-4": floats(O.ref_initial_condition("euler-sod-periodic", 4, "euler")),
               "heat-sine-1000-fnv": O.fnv1a64(O.ref_initial_condition("heat-sine", 1000))}
    g["dt_dx_sod"] = O.ref_finalize(O.RefConfig(equation="euler", grid_size=64, block_width=8))
    g["schedules"] = {f"{kind}-{w}-{h}": O.ref_schedule(kind, w, h) for kind in ("triangle", "diamond", "down")
                      for w, h in [(8, 1), (8, 2), (4, 1), (16, 1), (32, 2)]}
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json"), "w") as fh:
        json.dump(g, fh, indent=0)
    print("wrote golden.json")


if __name__ == "__main__":
    main()

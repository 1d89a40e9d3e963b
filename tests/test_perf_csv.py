"""CPU: measurement records, CSV, power-law fit and best_config of the B200
library (host-only) against the reference's own implementation
(src/perf.cpp, src/csv.cpp via oracle/_ref) and SPEC.md's acceptance
fixtures (Table 1 fit recovery); plus the C++ CLI on CPU."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

import paper_1811_08282_b200 as s1d
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1811_08282_b200", "_lib", "s1d")


FIELDS = ["equation", "method", "scheme", "mode", "grid_size", "block_width", "work_factor", "ranks", "steps",
          "avg_us_per_step", "setup_us", "messages_sent", "bytes_sent", "exchange_rounds", "virtual_comm_us"]


def ref_probe(req):
    """Run the reference's post-processing in a numpy-free subprocess."""
    import json
    import sys
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "ref_perf_probe.py")], input=json.dumps(req),
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    return json.loads(r.stdout)


def rec(eq=0, me=0, sc=1, n=1024, w=32, wf=0, r=2, T=50, mode=0, us=12.5, setup=3.25, msgs=10, by=160, rounds=5,
        vc=0.0):
    return s1d.TimingRecord(s1d.Equation(eq), s1d.Method(me), s1d.Scheme(sc), n, w, wf, r, T, s1d.Mode(mode), us,
                            setup, msgs, by, rounds, vc)


def to_ref(t):
    return [int(getattr(t, f)) if f in ("equation", "method", "scheme", "mode") else getattr(t, f) for f in FIELDS]


RECS = [rec(), rec(us=1.0 / 3.0, setup=1e-7), rec(eq=1, me=1, sc=0, n=1 << 20, w=1024, wf=3, r=8, T=6144,
                                                   us=123456.789012345, msgs=2 ** 40, by=2 ** 50, rounds=99999),
        rec(us=0.0, setup=0.0), rec(us=1e300, vc=2.5e-9), rec(mode=1, us=7.0)]

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="reference build not available")


def test_header():
    assert s1d.csv_header() == ("equation,method,scheme,n,w,wf,ranks,steps,mode,avg_us_per_step,msgs,bytes,rounds,"
                                "virtual_comm_us,setup_us")


@needs_ref
def test_csv_rows_match_reference():
    got = ref_probe({"records": [to_ref(t) for t in RECS]})
    assert [s1d.csv_row(t) for t in RECS] == got["rows"]


@needs_ref
def test_emit_csv_matches_reference_bytes(tmp_path):
    recs = RECS[::-1] + [rec(n=512), rec(w=16), rec(eq=1)]
    ours, theirs = tmp_path / "ours.csv", tmp_path / "ref.csv"
    s1d.emit_csv(recs, str(ours))
    got = ref_probe({"records": [to_ref(t) for t in recs], "emit_path": str(theirs)})
    assert got["emit_status"] == 0
    assert ours.read_bytes() == theirs.read_bytes()
    back = s1d.read_csv(str(ours))
    assert [s1d.csv_row(t) for t in back] == ours.read_text().splitlines()[1:]


def test_empty_csv_is_header_only(tmp_path):
    p = tmp_path / "e.csv"
    s1d.emit_csv([], str(p))
    assert p.read_text() == s1d.csv_header() + "\n"
    with pytest.raises(s1d.InvalidConfig):
        s1d.read_csv(str(tmp_path / "missing.csv"))


@pytest.mark.parametrize("A,b", [(1.33e-4, 0.937), (6.77e-3, 0.970), (2.0, 1.0), (0.5, 1.5)])
def test_power_law_fit_recovers_table1(A, b):
    # SPEC.md acceptance: Table 1 coefficients recovered from synthetic data
    ns = [5e5, 1e6, 5e6, 1e7]
    f = s1d.power_law_fit([(n, A * n ** b) for n in ns])
    assert abs(f.A - A) <= 1e-6 * A and abs(f.b - b) <= 1e-6 and f.r_squared >= 1 - 1e-12


@needs_ref
def test_power_law_fit_and_best_config_match_reference():
    rng = np.random.default_rng(3)
    cases = []
    for _ in range(10):
        xs = np.sort(rng.uniform(1e3, 1e8, 6))
        ys = 1e-3 * xs ** 0.9 * rng.uniform(0.9, 1.1, 6)
        cases.append([xs.tolist(), ys.tolist()])
    recs = [rec(w=64, us=10.0), rec(w=32, us=8.0), rec(w=16, wf=2, us=8.0), rec(w=16, wf=1, us=8.0)]
    got = ref_probe({"fits": cases, "records": [to_ref(t) for t in recs]})
    for (xs, ys), (st, A, b, r2) in zip(cases, got["fits"]):
        assert st == 0
        f = s1d.power_law_fit(list(zip(xs, ys)))
        assert (f.A, f.b, f.r_squared) == (A, b, r2)
    assert s1d.best_config(recs) is recs[got["best"]]


def test_power_law_fit_errors():
    with pytest.raises(s1d.DegenerateFit):
        s1d.power_law_fit([(10, 1), (10, 2), (10, 3)])
    with pytest.raises(s1d.InvalidConfig):
        s1d.power_law_fit([(10, 1), (20, 2)])


def test_best_config_tie_breaks():
    a, b, c = rec(w=64, us=10.0), rec(w=128, us=8.0), rec(w=64, us=8.0)
    assert s1d.best_config([a]) is a
    assert s1d.best_config([a, b]) is b
    assert s1d.best_config([b, c]) is c  # tie -> smaller w
    d, e = rec(w=64, wf=4, us=8.0), rec(w=64, wf=2, us=8.0)
    assert s1d.best_config([d, e]) is e  # then smaller WF
    assert s1d.speedup(10, 5) == 2.0 and s1d.flattening_speedup(3.4, 1.0) == 3.4


def test_cli_help_and_fit(tmp_path):
    assert subprocess.run([CLI, "--help"], capture_output=True).returncode == 0
    recs = [rec(n=n, w=w, us=1.33e-4 * n ** 0.937 * (1.0 if w == 64 else 1.5)) for n in (1 << 16, 1 << 18, 1 << 20)
            for w in (64, 128)]
    p = tmp_path / "t.csv"
    s1d.emit_csv(recs, str(p))
    out = subprocess.run([CLI, "fit", str(p)], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert "n^0.937" in out.stdout and "0.000133 " in out.stdout
    rep = subprocess.run([CLI, "report", str(p)], capture_output=True, text=True)
    assert rep.returncode == 0 and "swept" in rep.stdout


@pytest.mark.skipif(s1d.device_count() > 0, reason="GPU visible")
def test_cli_reports_no_device():
    r = subprocess.run([CLI, "solve", "n=64", "w=8"], capture_output=True, text=True)
    assert r.returncode == 1 and "status 22" in r.stderr

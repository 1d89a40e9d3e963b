"""CPU: the reference transport's message log (RunOptions::keep_message_log)
and per-rank counters (CommStats::per_rank), replayed by the library on the
host (s1d_message_log / s1d_rank_stats), equal the compiled reference's
(oracle/_ref) for both schemes, all equations, pads and WF; cf.
R/tests/test_decomp.cpp:147-199 (round and message counts)."""
import pytest

import paper_1811_08282_b200 as s1d
from oracle import oracle as O

EQ = {"heat": s1d.Equation.Heat, "euler": s1d.Equation.Euler}
ME = {"lengthening": s1d.Method.Lengthening, "flattening": s1d.Method.Flattening}
SC = {"swept": s1d.Scheme.Swept, "classic": s1d.Scheme.Classic}

CASES = [  # equation, method, scheme, n, w, ranks, wf, steps
    ("heat", "lengthening", "swept", 256, 16, 2, 0, 50),    # 6 cycles + 2 pad substeps
    ("heat", "lengthening", "classic", 96, 8, 3, 0, 7),
    ("heat", "lengthening", "swept", 320, 16, 3, 2, 21),
    ("euler", "lengthening", "swept", 256, 16, 2, 0, 13),
    ("euler", "flattening", "swept", 256, 16, 4, 0, 9),
    ("euler", "flattening", "classic", 128, 16, 2, 0, 3),
    ("heat", "lengthening", "swept", 64, 16, 2, 0, 3),      # no full cycle: pad only
]


@pytest.mark.skipif(not O.ref_available(), reason="compiled reference not available")
@pytest.mark.parametrize("case", CASES, ids=lambda c: "-".join(map(str, c)))
def test_message_log_and_per_rank_stats_equal_reference(case):
    eq, me, sc, n, w, ranks, wf, T = case
    ref = O.ref_run(O.RefConfig(equation=eq, method=me, scheme=sc, grid_size=n, block_width=w, ranks=ranks,
                                work_factor=wf, steps=T, mode="virtual", alpha=2e-6, beta=1e-9), keep_log=True)
    cfg = s1d.LaunchConfig(equation=EQ[eq], method=ME[me], scheme=SC[sc], grid_size=n, block_width=w, ranks=ranks,
                           work_factor=wf, steps=T)
    cfg.transport.alpha, cfg.transport.beta = 2e-6, 1e-9
    log = [(e.round, e.source, e.dest, e.tag, e.bytes) for e in s1d.message_log(cfg)]
    assert log == ref.log
    per = s1d.rank_stats(cfg)
    assert len(per) == ranks
    for r, st in enumerate(per):
        mine = [e for e in ref.log if e[1] == r]
        assert st.messages_sent == len(mine) and st.bytes_sent == sum(e[4] for e in mine)
        assert st.exchange_rounds == ref.exchange_rounds
        assert st.virtual_comm_time == ref.virtual_comm_time  # every rank joins every round
    assert sum(p.messages_sent for p in per) == ref.messages_sent
    assert sum(p.bytes_sent for p in per) == ref.bytes_sent

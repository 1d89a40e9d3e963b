"""CPU: invariants of the wavefront solve's issue order (host_wave.cpp via
s1d_debug_wave_schedule), the schedule engine.cu executes with CUDA streams,
events and, one process per GPU, the round flags of sync.cu.

Checked for many (chunks, head, tail, cycles), single- and multi-process:
  * every pipelined (phase, chunk) is issued exactly once, the middle once;
  * a chunk of phase p >= 1 follows chunks c-1, c, c+1 of phase p-1 (RAW on
    the edges it reads, WAR on the buffers their readers use); the first tail
    phase follows the middle, the middle follows every head chunk;
  * Up chunks in copy order;
  * multi-process: each pipelined phase signals its round once, in phase
    order, right after its last chunk; an end chunk (0 or K-1) of phase p
    follows the whole of phase p-1 and its signal, so a device wait for the
    neighbours' round p-1 never sits in front of this shard's own signal of
    p-1 (the deadlock-freedom argument of engine.cu wavefront_phases).
"""
import itertools

import pytest

import paper_1811_08282_b200 as s1d


def check(K, head, tail, cycles, xs):
    steps = s1d.wave_schedule(K, head, tail, cycles, xs)
    tail0 = cycles - tail
    phases = list(range(0, head + 1)) + list(range(tail0, cycles + 1))
    pos = {}
    middle = None
    signals = []
    for i, (kind, p, c) in enumerate(steps):
        if kind == "chunk":
            assert (p, c) not in pos, f"chunk {(p, c)} issued twice"
            assert p in phases and 0 <= c < K
            pos[(p, c)] = i
        elif kind == "signal":
            assert xs, "signals only between processes"
            signals.append((p, i))
        else:
            assert middle is None
            middle = i
    assert middle is not None
    assert set(pos) == {(p, c) for p in phases for c in range(K)}
    # Up chunks in copy order
    ups = [pos[(0, c)] for c in range(K)]
    assert ups == sorted(ups)
    for (p, c), i in pos.items():
        if p == 0:
            continue
        if p == tail0:
            assert i > middle
            continue
        for d in (-1, 0, 1):
            assert pos[(p - 1, (c + d) % K)] < i, f"{(p, c)} before its producer {(p - 1, (c + d) % K)}"
    for c in range(K):
        assert pos[(head, c)] < middle
    if xs:
        sig = dict((p, i) for p, i in signals)
        assert [p for p, _ in signals] == phases, "one signal per pipelined phase, in order"
        for p in phases:
            last = max(pos[(p, c)] for c in range(K))
            assert sig[p] == last + 1 or all(steps[j][0] == "signal" for j in range(last + 1, sig[p] + 1))
        for p in phases:
            if p == 0 or p == tail0:
                continue
            for c in (0, K - 1):
                assert sig[p - 1] < pos[(p, c)], f"end chunk {(p, c)} before the signal of phase {p - 1}"
    return steps


@pytest.mark.parametrize("xs", [False, True])
def test_wave_schedule_invariants(xs):
    n = 0
    for K, head, tail, extra in itertools.product([3, 4, 5, 7, 16, 32], [0, 1, 2, 3, 6], [0, 1, 2, 3], [0, 1, 5]):
        check(K, head, tail, head + tail + 2 + extra, xs)
        n += 1
    assert n > 300


def test_wave_schedule_overlaps_copies():
    # head Diamond chunks are interleaved with the Up chunks (they run while
    # later copies land), and the first Down chunk is issued before the tail
    # is complete (its copy-out starts early)
    steps = check(16, 2, 2, 48, False)
    order = [(p, c) for k, p, c in steps if k == "chunk"]
    first_d1 = next(i for i, (p, _) in enumerate(order) if p == 1)
    last_up = max(i for i, (p, _) in enumerate(order) if p == 0)
    assert first_d1 < last_up
    first_down = next(i for i, (p, _) in enumerate(order) if p == 48)
    last_tail = max(i for i, (p, _) in enumerate(order) if p == 47)
    assert first_down < last_tail


def test_wave_schedule_rejects_short_runs():
    with pytest.raises(s1d.InvalidConfig):
        s1d.wave_schedule(16, 3, 3, 7)
    with pytest.raises(s1d.InvalidConfig):
        s1d.wave_schedule(2, 1, 1, 10)

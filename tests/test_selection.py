"""The overlapping-section choice of the head frame — its host
half, on CPU: the product's `tracking.choose_sections` and the oracle's `select_sections` on
SPEC's worked examples and on random inputs (they are independent implementations and must
agree).  The device half (per-candidate visible counts) and the pre-track argmin are checked on
the GPU (`test_select_overlap_section_matches_oracle`)."""
import numpy as np

import oracle
from paper_2506_02741_b200.tracking import candidate_view_list, choose_sections


def _both(counts, nv, secs, gamma):
    a = choose_sections(counts, nv, secs, gamma)
    b = oracle.select_sections(counts, nv, secs, gamma)
    assert a == b, (a, b)
    return a


def test_spec_examples():
    # S:386 "exactly one frozen section → it is returned regardless of γ-filtering"
    assert _both([0, 0], 1000, [0, 0], 0.26) == [0]
    assert _both([900], 1000, [0], 0.26) == [0]
    # S:386 "two candidate sections where one views a disjoint region (zero visible fraction) →
    # the other is returned"
    assert _both([0, 800], 1000, [0, 1], 0.26) == [1]
    assert _both([800, 0], 1000, [0, 1], 0.26) == [0]
    # the most front (earliest) 3 sections containing a kept candidate
    assert _both([900, 10, 700, 800, 600, 500], 1000, [0, 1, 2, 3, 4, 5], 0.26) == [0, 2, 3]
    # γ is strict: exactly γ·n_valid visible does not pass
    assert _both([260, 261], 1000, [0, 1], 0.26) == [1]
    # several candidates per section count once
    assert _both([900, 900, 900, 900], 1000, [2, 2, 1, 1], 0.24) == [1, 2]
    # no valid pixel → nothing passes → the most recent section
    assert _both([0, 0, 0], 0, [0, 1, 2], 0.24) == [2]


def test_candidate_list_every_n1_frames():
    # P:180 "an overlap candidate view list with an interval of N1 frames", N1 = 5
    assert candidate_view_list(23) == [0, 5, 10, 15, 20]
    assert candidate_view_list(5) == [0]
    assert candidate_view_list(0) == []


def test_random_agreement():
    rng = np.random.default_rng(0)
    for _ in range(500):
        R = int(rng.integers(1, 20))
        nv = int(rng.integers(0, 5000))
        counts = [int(x) for x in rng.integers(0, nv + 1, R)]
        secs = sorted(int(x) for x in rng.integers(0, 8, R))
        _both(counts, nv, secs, float(rng.choice([0.24, 0.26, 0.5])))

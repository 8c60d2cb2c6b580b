"""Host-side logic of bench.py (no GPU): the useful-FLOP count of span layouts.

bench.py counts the visible (query, key) pairs of a span layout from the Fig. 10
rule at span level; here it is checked against the oracle's
per-pair enumeration, which the pins in test_oracle_pins.py tie to the paper.
"""
import numpy as np
import pytest

import bench
import oracle
import synth

pytestmark = pytest.mark.filterwarnings("ignore")


def _oracle_pairs(spans):
    tags = oracle.chunk_tags([s.chunk for s in spans], [s.kind for s in spans], [s.n_tokens for s in spans])
    n = len(tags[0])
    cnt = 0
    for i in range(n):
        for j in range(n):
            cnt += oracle.visible(int(tags[0][i]), int(tags[1][i]), int(tags[2][i]),
                                  int(tags[0][j]), int(tags[1][j]), int(tags[2][j]))
    return cnt


@pytest.mark.parametrize("layout", [
    synth.teacher_forcing_spans(3, 5),
    synth.teacher_forcing_spans(2, 7),
    [synth.Span(2, synth.CLEAN, 6), synth.Span(3, synth.CLEAN, 3), synth.Span(3, synth.NOISY, 5),
     synth.Span(4, synth.NOISY, 4), synth.Span(5, synth.CLEAN, 2)],
])
def test_visible_pairs_matches_oracle_enumeration(layout):
    assert bench.visible_pairs(layout) == _oracle_pairs(layout)


def test_teacher_forcing_fraction_fig10():
    # Fig. 10 worked example: [C0 C1 C2 Z1 Z2 Z3] x 64 tokens -> 61440 of 147456 pairs
    assert bench.visible_pairs(synth.teacher_forcing_spans(3, 64)) == 61440

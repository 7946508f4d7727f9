"""CPU check of the merge-round partition logic shared by the record tiers
(engine.cuh rec_round) and the global tier (chunk_round): a Python emulation
of G threads (tools/emulate_chunk.py) -- odd-length chunks over the round's
positions, pair search, merge-path split, dedupe at chunk starts, pair
crossing through the sentinels -- must reproduce Algorithm 1 exactly (oracle),
for group sizes that cut pairs at every kind of boundary."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import emulate_chunk as em  # noqa: E402
from inputs import random_sparse, stencil27, uniform_random  # noqa: E402


@pytest.mark.parametrize("G", [1, 3, 8, 32, 64])
@pytest.mark.parametrize("case", ["stencil", "random", "empties"])
def test_partition_reproduces_algorithm1(oracle_mod, G, case):
    if case == "stencil":
        A = B = stencil27(4, seed=1)
    elif case == "random":
        A = random_sparse(40, 60, 0.2, seed=7)
        B = random_sparse(60, 50, 0.3, seed=8)
    else:  # many empty B rows: empty lists and empty pairs everywhere
        A = random_sparse(30, 80, 0.25, seed=9)
        B = random_sparse(80, 40, 0.05, seed=10)
    ref, _ = oracle_mod.spgemm_brmerge(A, B)
    em.ROUND = em.chunk_round
    for r in range(A.rows):
        if A.rpt[r + 1] == A.rpt[r]:
            continue
        c, v = em.chunk_row(G, A, B, r)
        s, e = ref.rpt[r], ref.rpt[r + 1]
        assert list(ref.col[s:e]) == c, (G, r)
        np.testing.assert_array_equal(ref.val[s:e], np.array(v, dtype=np.float64))

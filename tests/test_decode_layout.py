"""Host descriptor layout of codec.decode_batch (CPU): the sort-free chain
order of _chain_layout against the direct definition — per stream, per plane
index, the frames from each intra frame up to the next, in frame order
(the dependency order of _reconstruct_plane, fk/codec.py:131-144)."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2602_09725_b200 import codec


def _reference(types_per_stream, hw):
    slots, chains = [], []
    k0 = 0
    for j, ft in enumerate(types_per_stream):
        n = len(ft)
        starts = [f for f in range(n) if ft[f] == 0]
        for a, b in zip(starts, starts[1:] + [n]):
            for p in range(3):
                if hw[j] > 0:
                    chains.append((len(slots), b - a, j))
                slots.extend(k0 + 3 * f + p for f in range(a, b))
        k0 += 3 * n
    return slots, chains


@pytest.mark.parametrize("seed", range(6))
def test_chain_layout_matches_definition(seed):
    rng = np.random.default_rng(seed)
    n_streams = int(rng.integers(1, 7))
    types = []
    for _ in range(n_streams):
        n = int(rng.integers(1, 40))
        ft = (rng.random(n) < 0.7).astype(np.uint8)   # 1 = inter
        ft[0] = 0                                     # every range starts intra
        types.append(ft)
    hw = rng.integers(0, 3, n_streams) * 64           # some empty planes
    dest, first, count, sid = codec._chain_layout(np.concatenate(types),
                                                  [len(t) for t in types], hw)
    slots, chains = _reference(types, hw)
    K = 3 * sum(len(t) for t in types)
    assert sorted(dest.tolist()) == list(range(K))
    order = np.empty(K, np.int64)
    order[dest] = np.arange(K)                        # plane k at slot dest[k]
    assert order.tolist() == slots
    assert list(zip(first.tolist(), count.tolist(), sid.tolist())) == chains


def test_split_parts_balances_bytes():
    assert codec._split_parts([0, 1, 2], [10, 10, 10]) == [[0, 1, 2]]   # below one part
    big = codec._PART_BYTES
    n = 2 * codec._MAX_PARTS
    parts = codec._split_parts(list(range(n)), [big] * n)
    assert [j for p in parts for j in p] == list(range(n))
    assert len(parts) == codec._MAX_PARTS and all(len(p) == 2 for p in parts)
    parts = codec._split_parts([3, 5], [5 * big, big])
    assert [j for p in parts for j in p] == [3, 5]

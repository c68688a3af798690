"""Pins for the oracle's KV-state rollback (Eq. 8-9)."""
import numpy as np
import pytest

import oracle as O


def _mask(lengths, cap):
    m = np.zeros((len(lengths), cap), np.uint8)
    for b, n in enumerate(lengths):
        m[b, :n] = 1
    return m


# ------------------------------------------------------------------ SPEC worked examples
def test_logical_rollback_spec_examples():
    m, L, f = O.rollback_mask(_mask([10], 10), 10, [3])
    assert m[0].sum() == 7 and L == 7 and list(m[0, 7:]) == [0, 0, 0]
    m, L, f = O.rollback_mask(_mask([10], 10), 10, [0])
    assert m[0].sum() == 10 and L == 10
    m, L, f = O.rollback_mask(_mask([10, 10, 10], 10), 10, [3, 1, 0])
    assert list(m.sum(1)) == [7, 9, 10]


def test_fix_kv_cache_spec_examples():
    # L' = (7, 9, 10), L = 10 -> no truncation
    m, L, _ = O.rollback_mask(_mask([7, 9, 10], 10), 10, [0, 0, 0])
    assert L == 10
    # L' = (8, 8, 8), L = 10 -> truncate to 8
    m, L, _ = O.rollback_mask(_mask([8, 8, 8], 10), 10, [0, 0, 0])
    assert L == 8
    # Eq. 9 with one command: r_min = min_b r_b trailing columns are reclaimed
    m, L, _ = O.rollback_mask(_mask([12, 12, 12], 12), 12, [5, 2, 3])
    assert L == 10 and list(m.sum(1)) == [7, 10, 9]


def test_rollback_overflow_flag():
    m, L, f = O.rollback_mask(_mask([4], 6), 6, [5])            # S:253 rollback-overflow
    assert f[0] & 8 and m[0].sum() == 4


def test_shadow_list_oracle_random_sequences():
    # attention_view (valid prefix) equals a plain shadow list under random
    # append / rollback / fix sequences; after fix, L = max_b L'_b.
    rng = np.random.default_rng(11)
    for trial in range(1000):
        B = int(rng.integers(1, 9))
        cap = 256
        mask = np.zeros((B, cap), np.uint8)
        toks = np.zeros((B, cap), np.int32)
        L = 0
        shadow = [[] for _ in range(B)]
        for step in range(int(rng.integers(1, 12))):
            k = int(rng.integers(1, 9))
            if L + k > cap:
                break
            # append with left-compaction: row b writes at its L'_b
            for b in range(B):
                n = int(mask[b].sum())
                new = rng.integers(0, 1000, k)
                toks[b, n:n + k] = new
                mask[b, n:n + k] = 1
                mask[b, n + k:] = 0
                shadow[b].extend(int(t) for t in new)
            L = max(L, int(mask.sum(1).max()))
            r = np.array([rng.integers(0, int(mask[b].sum()) + 1) for b in range(B)], np.int32)
            mask, L, f = O.rollback_mask(mask, L, r)
            assert not f.any()
            for b in range(B):
                if r[b]:
                    del shadow[b][len(shadow[b]) - int(r[b]):]
                n = int(mask[b].sum())
                assert mask[b, :n].all() and not mask[b, n:].any()        # prefix-valid
                assert list(toks[b, :n]) == shadow[b]                     # attention view
            assert L == max(len(s) for s in shadow)


# ------------------------------------------------------------------ paged view
def _paged_state(rng, B, bs, max_len):
    max_blocks = (max_len + bs - 1) // bs
    seq = rng.integers(0, max_len + 1, B).astype(np.int32)
    pool = B * max_blocks
    perm = rng.permutation(pool).astype(np.int32)
    bt = np.full((B, max_blocks), -1, np.int32)
    off = 0
    for b in range(B):
        n = (int(seq[b]) + bs - 1) // bs
        bt[b, :n] = perm[off:off + n]
        off += n
    free = np.full(pool, -1, np.int32)
    free[:pool - off] = perm[off:]
    return seq, bt, free, pool - off, pool


def test_paged_rollback_conserves_blocks_and_matches_mask_view():
    rng = np.random.default_rng(5)
    for trial in range(300):
        B, bs, max_len = int(rng.integers(1, 16)), 16, int(rng.integers(1, 300))
        seq, bt, free, nfree, pool = _paged_state(rng, B, bs, max_len)
        r = np.array([rng.integers(0, s + 1) for s in seq], np.int32)
        mask = _mask(seq, max_len)
        o = O.rollback_paged(seq, bt, bs, free, nfree, r, cache_mask=mask)
        assert not o["flags"].any()
        assert (o["seq_len"] == seq - r).all()
        held = o["block_table"][o["block_table"] >= 0]
        freed = o["free_ids"][:o["free_count"]]
        allids = np.concatenate([held, freed])
        assert allids.size == pool and np.unique(allids).size == pool        # conservation
        for b in range(B):
            need = (int(o["seq_len"][b]) + bs - 1) // bs
            assert (o["block_table"][b, :need] == bt[b, :need]).all()
            assert (o["block_table"][b, need:] == -1).all()
            assert o["cache_mask"][b].sum() == o["seq_len"][b]               # paged == mask view
        # deterministic release order: request-major, ascending block index
        expect = []
        for b in range(B):
            j0 = (int(seq[b] - r[b]) + bs - 1) // bs
            j1 = (int(seq[b]) + bs - 1) // bs
            expect.extend(bt[b, j0:j1])
        assert list(freed[nfree:]) == expect


def test_paged_rollback_overflow_and_freelist_flags():
    seq = np.array([20, 5], np.int32)
    bt = np.array([[0, 1], [2, -1]], np.int32)
    free = np.full(4, -1, np.int32)
    o = O.rollback_paged(seq, bt, 16, free, 0, np.array([17, 6], np.int32))
    assert o["flags"][1] & 8 and o["seq_len"][1] == 5          # r > seq_len: untouched
    assert o["seq_len"][0] == 3 and o["free_count"] == 1 and o["free_ids"][0] == 1
    free = np.full(1, -1, np.int32)
    o = O.rollback_paged(np.array([40], np.int32), np.array([[0, 1, 2]], np.int32), 16, free, 0,
                         np.array([39], np.int32))
    assert o["flags"][0] & 16 and o["seq_len"][0] == 1 and (o["block_table"] == [[0, 1, 2]]).all()


def test_paged_rollback_rejects_a_length_beyond_the_block_table_row():
    # DESIGN.md R22: a sequence longer than its block-table row can hold is an inconsistent
    # caller state; the request is left untouched and flagged, the others proceed
    bt = np.arange(2 * 3, dtype=np.int32).reshape(2, 3)          # 3 blocks of 4 tokens per row
    o = O.rollback_paged(np.array([13, 9]), bt, 4, np.full(8, -1, np.int32), 0, np.array([2, 5]))
    assert o["seq_len"].tolist() == [13, 4] and o["flags"][0] != 0 and o["flags"][1] == 0
    assert o["block_table"][0].tolist() == [0, 1, 2]                   # untouched
    assert o["block_table"][1].tolist() == [3, -1, -1] and o["free_count"] == 2
    assert o["free_ids"][:2].tolist() == [4, 5]

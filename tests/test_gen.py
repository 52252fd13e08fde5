"""Input generator checks (CPU): determinism, shard consistency, table structure."""
import numpy as np

import gen


def test_deterministic_and_shard_consistent():
    c = gen.CONFIGS["c2"]
    full = gen.store_emb(c.store_seed, 20_000, c.dim)
    again = gen.store_emb(c.store_seed, 20_000, c.dim)
    np.testing.assert_array_equal(full, again)
    for world in (2, 3, 8):
        parts = []
        for r in range(world):
            off, n = gen.shard_range(20_000, world, r)
            parts.append(gen.store_emb(c.store_seed, 20_000, c.dim, off, n))
        np.testing.assert_array_equal(np.concatenate(parts), full)
    a_full = gen.store_act(c.store_seed, 20_000, c.layers, c.experts, c.moe_topk)
    off, n = gen.shard_range(20_000, 4, 3)
    np.testing.assert_array_equal(
        gen.store_act(c.store_seed, 20_000, c.layers, c.experts, c.moe_topk, off, n),
        a_full[off:off + n])


def test_shard_range_tiles():
    for n_total in (1, 7, 1000, 10_000_000):
        for world in (1, 2, 3, 4, 8):
            covered = 0
            for r in range(world):
                off, n = gen.shard_range(n_total, world, r)
                assert off == covered or n == 0
                covered += n
            assert covered == n_total


def test_activation_rows_are_frequencies():
    """s~ = frec / sum_k frec: rows sum to 1, entries in [0,1], and
    each row is count/total for integer counts with total <= N_in*topk*1.5."""
    for name in ("tiny", "c2", "c3"):
        c = gen.CONFIGS[name]
        a = gen.store_act(c.store_seed, c.n, c.layers, c.experts, c.moe_topk, 0, 500)
        assert a.dtype == np.float32 and np.all(a >= 0) and np.all(a <= 1)
        np.testing.assert_allclose(a.sum(-1), 1.0, atol=c.experts * 2 ** -23)
        # smallest nonzero entry times the total is an integer count
        nz = a[a > 0]
        assert nz.min() >= 1.0 / (256 * 1.5 * c.moe_topk) - 1e-9


def test_embeddings_are_clustered():
    """Intra-cluster cosine clearly exceeds inter-cluster cosine."""
    c = gen.CONFIGS["c3"]
    n = 3000
    x = gen.bf16_bits_to_f32(gen.store_emb(c.store_seed, c.n, c.dim, 0, n)).astype(np.float64)
    cl = np.array([gen.cluster_of(c.store_seed, c.n, j) for j in range(n)])
    xn = x / np.linalg.norm(x, axis=1, keepdims=True)
    s = xn @ xn.T
    same = cl[:, None] == cl[None, :]
    np.fill_diagonal(same, False)
    inter = ~same
    np.fill_diagonal(inter, False)
    assert same.sum() > 100
    assert s[same].mean() > 0.3 and abs(s[inter].mean()) < 0.02


def test_query_mix():
    c = gen.CONFIGS["tiny"]
    x = gen.store_emb(c.store_seed, c.n, c.dim)
    q = gen.queries(c.store_seed, c.query_seed, c.n, c.dim, 24, mode=1)
    for i in range(24):
        src = gen.query_source_row(c.query_seed, c.n, i, mode=1)
        if i % 8 in (4, 5):
            np.testing.assert_array_equal(q[i], x[src])
        elif i % 8 == 6:
            assert not np.array_equal(q[i], x[src])
        elif i % 8 == 7:
            np.testing.assert_array_equal(q[i], q[i - 1])
        else:
            assert src == -1
    q0 = gen.queries(c.store_seed, c.query_seed, c.n, c.dim, 24, mode=0)
    np.testing.assert_array_equal(q0[:4], q[:4])


def test_bf16_helpers_roundtrip():
    v = np.array([1.0, -2.5, 0.0, 3.140625, 1e-3], np.float32)
    b = gen.f32_to_bf16_bits(v)
    np.testing.assert_array_equal(gen.bf16_bits_to_f32(b)[:4], v[:4])

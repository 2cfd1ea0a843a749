"""Input generator: determinism and calibration against the graph-size table
(PAPER.md `tab:graph_table` P:302-322)."""
import numpy as np

from paper_2411_15997_b200 import tracegen as G


def test_deterministic():
    a = G.generate("c1")
    b = G.generate("c1")
    for k in G.FIELDS:
        assert (a[k] == b[k]).all()


def test_graph_size_calibration():
    tr = G.generate(dict(G.CONFIGS["c2"], n_calls=400_000, n_users=200, seed=5))
    meta = tr["meta"].astype(np.int64)
    heads = ((meta >> 8) & 255) == 1
    m = (meta >> 16) & 255
    m = m[heads]
    assert len(m) > 100_000
    for lo, hi, pct in G.GRAPH_BUCKETS:
        f = 100.0 * ((m >= lo) & (m <= hi)).mean()
        assert abs(f - pct) <= 2.0, (lo, hi, f, pct)


def test_trace_shape():
    tr = G.generate("c1")
    assert tr["n_calls"] == 200 and tr["n_users"] == 4 and tr["n_apps"] == 2
    tiers = np.unique(tr["meta"] >> 24)
    assert (tiers > 0).sum() == 1          # exactly one abusive user's tier
    assert (np.diff(tr["t_ms"].astype(np.int64)) >= 0).all()


def test_shards_partition_users():
    tr = G.generate(dict(G.CONFIGS["c2"], n_calls=5000, n_users=50, seed=9))
    parts = [G.shard_by_user(tr, r, 4) for r in range(4)]
    assert sum(p["n_calls"] for p in parts) == tr["n_calls"]
    users = [set(np.unique(p["user"])) for p in parts]
    for i in range(4):
        for j in range(i + 1, 4):
            assert not (users[i] & users[j])

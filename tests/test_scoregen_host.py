"""Score-generator host logic (no GPU): kind names (score_gen.cpp:27-44),
config defaults (score_gen.hpp:29-52), the C struct, and the oracle's
generator sanity (rows on the simplex, deterministic per (seed, step, layer,
token))."""
import numpy as np
import pytest

import oracle
from paper_2511_02237_b200 import routing as R
from paper_2511_02237_b200 import scoregen as G


def test_kind_names():
    for k, name in ((G.GenKind.Dirichlet, "dirichlet"), (G.GenKind.Clustered, "clustered"),
                    (G.GenKind.Replay, "replay")):
        assert G.to_string(k) == name and G.gen_kind_from_string(name) == k
    with pytest.raises(R.InvalidArgument, match="unknown score generator 'gauss'"):
        G.gen_kind_from_string("gauss")


def test_defaults_and_c_struct():
    c = G.ScoreGenConfig()
    assert (c.kind, c.n_experts, c.batch, c.steps, c.layers, c.seed) == (G.GenKind.Dirichlet, 128, 16, 1, 1, 0)
    assert (c.alpha, c.groups, c.within_group_concentration, c.between_group_spread) == (1.0, 2, 4.0, 2.0)
    s = G.ScoreGenConfig(G.GenKind.Clustered, 64, 8, 3, 2, 2 ** 64 - 1, 0.5, 4, 2.0, 1.5).to_c()
    assert (s.kind, s.n_experts, s.batch, s.steps, s.layers, s.seed, s.groups) == (1, 64, 8, 3, 2, 2 ** 64 - 1, 4)
    with pytest.raises(R.InvalidArgument, match="replay"):
        G.ScoreGenConfig(G.GenKind.Replay, trace_path="x").to_c()


def test_oracle_generators_sane():
    d = oracle.gen_dirichlet(32, 6, 9, 0.3, 1, 2)
    assert np.allclose(d.sum(axis=1), 1.0) and (d >= 0).all()
    assert np.array_equal(d, oracle.gen_dirichlet(32, 6, 9, 0.3, 1, 2))
    assert not np.array_equal(d, oracle.gen_dirichlet(32, 6, 9, 0.3, 2, 2))
    # token i's row does not depend on the batch size (streams keyed per token)
    assert np.array_equal(d[:4], oracle.gen_dirichlet(32, 4, 9, 0.3, 1, 2))
    c = oracle.gen_clustered(32, 6, 9, 2, 4.0, 0.0, 0, 0)
    assert np.allclose(c, 1.0 / 32)

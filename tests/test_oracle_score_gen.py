"""The oracle's restated score generators (oracle/oea_oracle.c) are the
compiled reference's gen_scores (score_gen.cpp:100-160) bit for bit."""
import numpy as np
import pytest

import oracle


@pytest.mark.skipif(not oracle.reference_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("alpha", [0.05, 0.3, 1.0, 2.5])
def test_dirichlet_restatement_pinned(alpha):
    R = oracle.Reference()
    for step, layer in ((0, 0), (3, 5)):
        ref = R.gen_scores("dirichlet", 128, 16, 42, step, layer, alpha=alpha)
        assert np.array_equal(ref, oracle.gen_dirichlet(128, 16, 42, alpha, step, layer))


@pytest.mark.skipif(not oracle.reference_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("groups,conc,spread", [(1, 4.0, 2.0), (3, 0.5, 5.0), (2, 4.0, 0.0)])
def test_clustered_restatement_pinned(groups, conc, spread):
    R = oracle.Reference()
    ref = R.gen_scores("clustered", 64, 10, 7, 2, 1, groups=groups, conc=conc, spread=spread)
    assert np.array_equal(ref, oracle.gen_clustered(64, 10, 7, groups, conc, spread, 2, 1))

"""Error behaviour of the GPU path that the reference specifies
(SURVEY §8(b) Errors): the per-layer non-finite feature check
(potential.cpp:107-115, called per conv layer at :772 inside
parallel_for_partitions, whose wrapper is engine.cpp:278-283) and parameter
validation (potential.cpp:150-176)."""
import numpy as np
import pytest

from paper_2506_02023_b200 import graphmd as G
from tests import systems as S

pytestmark = pytest.mark.gpu


def overflow_params(F=16, r3=0.0):
    """Oxygen embeddings beyond the fp32 range: h0 = inf on every O row, so
    every atom's layer-0 feature is non-finite (the fp32 features overflow;
    the check reports it instead of returning a non-finite energy)."""
    prm = G.ToyPotentialParams.init(3, F, 8, 2, 5.0, r3)
    prm.embedding.reshape(119, F)[8] = 1e300
    return prm


@pytest.mark.parametrize("p", [1, 2, 4])
@pytest.mark.parametrize("F", [16, 24])
def test_nonfinite_feature_reports_first_row(p, F):
    s = S.quartz((3, 3, 3))
    d = G.Distributed.create_distributed(s, 5.0, None, p, 1, True)
    first = int(d.atom_parts().parts[0].layout.node_array[0]) if p > 1 else 0
    with pytest.raises(G.Error, match=rf"^worker for partition 0 failed: non-finite feature at "
                                      rf"layer 0, atom {first}$"):
        G.forward_distributed(d, overflow_params(F))
    # the handle stays usable
    out = G.forward_distributed(d, G.ToyPotentialParams.init(3, F, 8, 2, 5.0))
    assert np.isfinite(out.energy)


def test_nonfinite_feature_rank_group():
    s = S.quartz((3, 3, 4))
    hs = G.local_group(2)
    prm = overflow_params()

    def rank(r):
        def go():
            d = G.Distributed.create_distributed(s, 5.0, None, 2, 1, True, handle=hs[r])
            try:
                G.forward_distributed(d, prm)
            except G.Error as e:
                return str(e)
            return None
        return go

    msgs = G.run_ranks([rank(r) for r in range(2)])
    assert msgs[0] is not None and msgs[0] == msgs[1]
    assert msgs[0].startswith("worker for partition 0 failed: non-finite feature at layer 0, atom ")


def test_nonfinite_parameter_names_the_array():
    prm = G.ToyPotentialParams.init(1, 16, 8, 2, 5.0)
    prm.w3[0] = np.inf
    with pytest.raises(G.Error, match="parameter array w3 contains a non-finite value"):
        prm.validate()

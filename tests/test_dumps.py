"""Graph / plan dump formats: AtomGraph::dump_csv,
PartitionedLineGraph::dump_csv and partition_plan_to_json of the GPU path are
byte-identical to the reference's own dumps (oracle/_ref) of the same system,
so large-scale golden diffs need nothing but `cmp`."""
import pytest

from paper_2506_02023_b200 import graphmd as G
from tests import systems as S



@pytest.mark.parametrize("p", [1, 2, 4])
def test_json_layout_pinned_to_reference(oracle_ref, p):
    """The plan JSON writer reproduces the reference's layout byte for byte
    (checked on the reference's own output; no GPU needed)."""
    import json
    s = S.quartz((2, 2, 3))
    js = oracle_ref.create(*S.as_args(s), 5.0, p=p, allow_narrow=True).plan_json()
    assert G._json_dump2(json.loads(js), 0) == js


@pytest.mark.gpu
@pytest.mark.parametrize("p", [1, 3])
def test_dumps_identical_to_reference(tmp_path, oracle_ref, p):
    s = S.quartz((3, 3, 3))
    d = G.Distributed.create_distributed(s, 5.0, 3.0, p, 1, True)
    ref = oracle_ref.create(*S.as_args(s), 5.0, r3=3.0, p=p, allow_narrow=True)
    d.graph().dump_csv(str(tmp_path / "g.csv"))
    ref.dump_graph(str(tmp_path / "g_ref.csv"))
    assert (tmp_path / "g.csv").read_bytes() == (tmp_path / "g_ref.csv").read_bytes()
    d.line_parts().dump_csv(str(tmp_path / "l.csv"))
    ref.dump_line(str(tmp_path / "l_ref.csv"))
    assert (tmp_path / "l.csv").read_bytes() == (tmp_path / "l_ref.csv").read_bytes()
    assert G.partition_plan_to_json(d.atom_parts()) == ref.plan_json()


@pytest.mark.gpu
@pytest.mark.parametrize("p", [1, 3])
def test_cpp_header_dumps_identical_to_reference(tmp_path, oracle_ref, p):
    """The same three dumps written through include/graphmd_b200/graphmd.hpp."""
    import subprocess

    from tests.test_cpp import BIN, build
    build()
    r = subprocess.run([BIN, "--dump", str(tmp_path), str(p)], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    s = S.quartz((3, 3, 3))  # = random_perturb(make_supercell(quartz, 3x3x3), 0.05, 1)
    ref = oracle_ref.create(*S.as_args(s), 5.0, r3=3.0, p=p, allow_narrow=True)
    ref.dump_graph(str(tmp_path / "g_ref.csv"))
    ref.dump_line(str(tmp_path / "l_ref.csv"))
    assert (tmp_path / "g.csv").read_bytes() == (tmp_path / "g_ref.csv").read_bytes()
    assert (tmp_path / "l.csv").read_bytes() == (tmp_path / "l_ref.csv").read_bytes()
    assert (tmp_path / "plan.json").read_text() == ref.plan_json()

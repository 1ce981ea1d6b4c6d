"""The audit / bench / md harness (the reference driver's
commands, proj/tools/graphmd_cli.cpp, and CSV schemas, proj/docs/formats.md:
40-78).  CPU: option and configuration errors (exit 2).  GPU: audit passes
(partitioned bitwise == one partition) and fails under the corrupt-plan
hook, every bench mode writes its schema, md --paired agrees."""
import io
import os

import pytest

from paper_2506_02023_b200 import harness as H

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
QUARTZ = os.path.join(ROOT, "tests", "golden", "quartz.xyz")

SCHEMAS = {  # formats.md:40-78
    "strong": "mode,p,threads,atoms,edges,time_s,baseline_s,normalized",
    "weak": "mode,p,threads,atoms,edges,time_s,baseline_s,normalized",
    "capacity": "budget_bytes,scale,atoms,estimated_bytes,status,time_s",
    "density": "density_factor,atoms,edges,time_s",
    "breakdown": "p,atoms,graph_creation_s,feature_calculation_s,forward_pass_s,backward_pass_s,total_s",
}


def test_config_errors_exit_2(tmp_path):
    assert H.main(["audit"]) == H.EXIT_CONFIG  # --fixture is required
    assert H.main(["audit", "--fixture", str(tmp_path / "missing.xyz")]) == H.EXIT_CONFIG
    assert H.main(["bench", "--fixture", QUARTZ, "--mode", "sideways"]) == H.EXIT_CONFIG
    assert H.main(["audit", "--fixture", QUARTZ, "--reps", "2,2"]) == H.EXIT_CONFIG
    assert H.main(["md", "--fixture", QUARTZ, "--dt", "-1"]) == H.EXIT_CONFIG


def test_capacity_estimate_scales_with_atoms():
    s = H.Setup(QUARTZ, (2, 2, 2)).system()
    big = H.Setup(QUARTZ, (4, 4, 4)).system()
    p = H.Setup(QUARTZ).params()
    assert 7.5 < H.estimate_bytes(big, p, 1) / H.estimate_bytes(s, p, 1) < 8.5


@pytest.mark.gpu
def test_audit_passes_and_catches_a_corrupt_plan():
    out, err = io.StringIO(), io.StringIO()
    setup = H.Setup(QUARTZ, (3, 3, 3), (1, 2, 3), allow_narrow=True, threebody_cutoff=3.0)
    assert H.audit(setup, out=out, err=err) == H.EXIT_OK, err.getvalue()
    for line in out.getvalue().splitlines():  # partitioned == one partition, bitwise
        assert line.endswith("max|dE|/atom=0 max|dF|=0 max|dS|=0"), line
    out, err = io.StringIO(), io.StringIO()
    assert H.audit(setup, corrupt_plan=True, out=out, err=err) in (H.EXIT_TOLERANCE, H.EXIT_RUNTIME)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", sorted(SCHEMAS))
def test_bench_modes_write_the_reference_schemas(mode, tmp_path):
    path = tmp_path / f"{mode}.csv"
    setup = H.Setup(QUARTZ, (3, 3, 3), (1, 2), allow_narrow=True, cutoff=4.0)
    rc = H.bench(setup, mode, repeat=3, keep_last=2, budget_bytes=64 << 20, densities=(0.8, 1.0),
                 out_path=str(path))
    assert rc == H.EXIT_OK
    lines = path.read_text().splitlines()
    assert lines[0] == SCHEMAS[mode]
    rows = [ln.split(",") for ln in lines[1:]]
    assert len(rows) == {"capacity": 1, "density": 2}.get(mode, 2)
    assert all(len(r) == len(lines[0].split(",")) for r in rows)
    if mode == "breakdown":
        for r in rows:
            parts = [float(x) for x in r[2:6]]
            assert all(x > 0 for x in parts) and abs(sum(parts) - float(r[6])) < 1e-9
    if mode == "capacity":
        assert rows[0][4] == "ok" and int(rows[0][3]) <= 64 << 20
    if mode == "weak":
        assert int(rows[1][3]) == 2 * int(rows[0][3])  # replicated along a


@pytest.mark.gpu
def test_md_paired_run(tmp_path):
    out = io.StringIO()
    setup = H.Setup(QUARTZ, (2, 2, 2), (2,), allow_narrow=True)
    csv = tmp_path / "e.csv"
    rc = H.md(setup, 5, dt=0.5, out_path=str(csv), paired=True, pair_tol=1e-9, out=out)
    assert rc == H.EXIT_OK, out.getvalue()
    assert "paired max|dx|=0 " in out.getvalue()
    assert len(csv.read_text().splitlines()) == 1 + 6

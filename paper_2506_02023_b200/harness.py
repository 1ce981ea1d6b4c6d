"""Audit and benchmark harness of the B200 path: the
reference command-line driver's `audit`, `bench` and `md` commands
(proj/tools/graphmd_cli.cpp:70-126, 137-295, 299-355) re-expressed over the
GPU library, writing the reference's CSV schemas (proj/docs/formats.md:40-78)
and using its exit codes (formats.md "CLI exit codes").

    python -m paper_2506_02023_b200.harness audit --fixture tests/golden/quartz.xyz --reps 4,4,4
    python -m paper_2506_02023_b200.harness bench --fixture ... --mode breakdown --partitions 1,2,4
    python -m paper_2506_02023_b200.harness md --fixture ... --steps 100 --paired

Differences from the CPU driver, all following from the device:
* timings are the library's CUDA-event StepTiming (graph creation measured on
  the device, not by a host clock around create_distributed);
* `audit` compares each partition count with the one-partition evaluation on
  the same GPU (the fp64 serial evaluator is the test oracle, not shipped);
  partitioned results are bitwise those of p = 1, so any
  deviation at all is reported, and the tolerances default to the fp32
  contract of tests/conftest.py;
* `threads` is accepted and written to the CSVs but not used (one GPU);
* `capacity` estimates the device footprint of this implementation
   against a budget that defaults to the free device memory.
"""
from __future__ import annotations

import argparse
import ctypes as C
import io
import math
import sys
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import graphmd as G

EXIT_OK, EXIT_TOLERANCE, EXIT_CONFIG, EXIT_RUNTIME = 0, 1, 2, 3


@dataclass
class Setup:
    """The driver's common options (graphmd_cli.cpp:28-37 defaults)."""
    fixture: str = ""
    reps: Sequence[int] = (1, 1, 1)
    partitions: Sequence[int] = (1, 2, 4)
    threads: int = 0
    cutoff: float = 4.0
    threebody_cutoff: float = 0.0
    seed: int = 12345
    allow_narrow: bool = False
    device: int = 0

    def system(self) -> G.AtomicSystem:
        s = G.load_xyz(self.fixture)
        if tuple(self.reps) != (1, 1, 1):
            s = G.make_supercell(s, tuple(self.reps))
        return s

    def params(self) -> G.ToyPotentialParams:
        return G.ToyPotentialParams.init(self.seed, 16, 8, 2, self.cutoff, self.threebody_cutoff)


def _evaluate(system: G.AtomicSystem, params: G.ToyPotentialParams, p: int, allow_narrow: bool,
              device: int, handle: Optional[G._Handle] = None):
    """create_distributed + forward_distributed with all four StepTiming
    categories from the library's events; returns (output, timing, edges)."""
    r3 = params.r_3body if params.threebody() else None
    d = G.Distributed.create_distributed(system, params.r_atom, r3, p, 1, allow_narrow,
                                         device=device, handle=handle)
    h = d.handle
    L = G.lib()
    h.check(L.gmd_set_params(h.h, params.feature_width, params.basis_count, params.layers,
                             params.r_atom, params.r_3body, G._p(params.blob)))
    n = d.num_nodes()
    e = C.c_double()
    pa, fo, st, tm = np.zeros(n), np.zeros((n, 3)), np.zeros(9), np.zeros(4)
    h.check(L.gmd_forward(h.h, C.byref(e), G._p(pa), G._p(fo), G._p(st), G._p(tm), 0))
    t = G.StepTiming(*tm)
    return G.PotentialOutput(e.value, pa, fo, st.reshape(3, 3)), t, d.num_edges()


@dataclass
class TimedRun:
    mean: G.StepTiming = field(default_factory=G.StepTiming)
    time_s: float = 0.0
    atoms: int = 0
    edges: int = 0


def time_evaluation(system: G.AtomicSystem, params: G.ToyPotentialParams, p: int, allow_narrow: bool,
                    repeat: int, keep_last: int, device: int = 0) -> TimedRun:
    """The driver's protocol (graphmd_cli.cpp:137-168): `repeat` evaluations,
    the mean StepTiming of the last `keep_last`.  The device buffers are
    reused across repetitions (one handle), as in an MD run."""
    if repeat < 1 or keep_last < 1 or keep_last > repeat:
        raise G.Error("need repeat >= keep-last >= 1")
    h = G._Handle(device)
    kept: List[G.StepTiming] = []
    run = TimedRun(atoms=system.size())
    for r in range(repeat):
        _, t, ne = _evaluate(system, params, p, allow_narrow, device, h)
        run.edges = ne
        if r >= repeat - keep_last:
            kept.append(t)
    for t in kept:
        run.mean += t
    k = 1.0 / len(kept)
    run.mean = G.StepTiming(run.mean.graph_creation * k, run.mean.feature_calculation * k,
                            run.mean.forward_pass * k, run.mean.backward_pass * k)
    run.time_s = run.mean.total()
    return run


def estimate_bytes(system: G.AtomicSystem, params: G.ToyPotentialParams, p: int) -> int:
    """Device footprint of one evaluation: per edge the slab key
    (8 B), src / packed image / (v, d) / d / bond flag (29 B), local source and
    three-body tables (~12 B); per atom the positions and search arrays
    (~150 B) and (L + 4) feature rows of F floats; per partition a plan."""
    n = system.size()
    vol = max(1e-9, abs(np.linalg.det(system.lattice)))
    degree = 4.0 / 3.0 * math.pi * params.r_atom ** 3 * n / vol
    edges = int(degree * n) + n
    F = params.feature_width
    per_edge = 8 + 29 + 12
    per_atom = 150 + 4 * F * (params.layers + 4) + 32
    return edges * per_edge + n * per_atom + p * 4096


def audit(setup: Setup, tol_energy: float = 2e-5, tol_force: float = 2e-4, tol_stress: float = 2e-6,
          corrupt_plan: bool = False, out=sys.stdout, err=sys.stderr) -> int:
    """graphmd_cli.cpp:70-126 over the GPU: every partition count against the
    one-partition evaluation.  Exit 0 / 1 (tolerance) / 2 (config) / 3 (runtime)."""
    try:
        system, params = setup.system(), setup.params()
    except Exception as e:  # unreadable fixture, bad widths
        print(f"config error: {e}", file=err)
        return EXIT_CONFIG
    try:
        ref, _, _ = _evaluate(system, params, 1, setup.allow_narrow, setup.device)
        ok = True
        for p in setup.partitions:
            r3 = params.r_3body if params.threebody() else None
            d = G.Distributed.create_distributed(system, params.r_atom, r3, p, setup.threads,
                                                 setup.allow_narrow, device=setup.device)
            if corrupt_plan:
                d.corrupt_transfer_plan_for_test()
            o = G.forward_distributed(d, params)
            de = float(np.abs(o.per_atom - ref.per_atom).max())
            df = float(np.abs(o.forces - ref.forces).max())
            ds = float(np.abs(o.stress - ref.stress).max())
            print(f"p={p} max|dE|/atom={de:.6g} max|dF|={df:.6g} max|dS|={ds:.6g}", file=out)
            for what, v, tol in (("energy", de, tol_energy), ("force", df, tol_force),
                                 ("stress", ds, tol_stress)):
                if not v <= tol:
                    print(f"FAIL p={p} {what} {v:.6g} > {tol:.6g}", file=err)
                    ok = False
        return EXIT_OK if ok else EXIT_TOLERANCE
    except Exception as e:
        print(f"runtime error: {e}", file=err)
        return EXIT_RUNTIME


def _csv_num(x) -> str:
    return format(x, ".9g") if isinstance(x, float) else str(x)


def bench(setup: Setup, mode: str, repeat: int = 20, keep_last: int = 10, budget_bytes: int = 0,
          densities: Sequence[float] = (0.5, 1.0, 2.0), out_path: str = "", out=sys.stdout,
          err=sys.stderr) -> int:
    """graphmd_cli.cpp:184-295: strong / weak / capacity / density /
    breakdown CSVs in the reference's schemas (formats.md:40-78)."""
    try:
        if mode not in ("strong", "weak", "capacity", "density", "breakdown"):
            raise G.Error(f"unknown bench mode: {mode}")
        base, params = setup.system(), setup.params()
    except Exception as e:
        print(f"config error: {e}", file=err)
        return EXIT_CONFIG
    try:
        rows: List[List] = []
        run: Callable[[G.AtomicSystem, int], TimedRun] = lambda s, p: time_evaluation(
            s, params, p, setup.allow_narrow, repeat, keep_last, setup.device)
        thr = lambda p: setup.threads if setup.threads > 0 else p
        if mode in ("strong", "weak"):
            header = "mode,p,threads,atoms,edges,time_s,baseline_s,normalized"
            baseline = time_evaluation(base, params, 2, setup.allow_narrow, repeat, keep_last, setup.device)
            for p in setup.partitions:
                s = G.make_supercell(base, (p, 1, 1)) if (mode == "weak" and p > 1) else base
                r = run(s, p)
                norm = ((r.time_s / r.atoms) / (baseline.time_s / baseline.atoms) if mode == "weak"
                        else r.time_s / baseline.time_s)
                rows.append([mode, p, thr(p), r.atoms, r.edges, r.time_s, baseline.time_s, norm])
        elif mode == "capacity":
            header = "budget_bytes,scale,atoms,estimated_bytes,status,time_s"
            p0 = setup.partitions[0]
            if budget_bytes <= 0:
                import torch
                budget_bytes = int(torch.cuda.mem_get_info(setup.device)[0])
            fits = lambda k: estimate_bytes(G.make_supercell(base, (k, k, k)), params, p0) <= budget_bytes
            if not fits(1):
                rows.append([budget_bytes, 1, base.size(), estimate_bytes(base, params, p0), "exceeded", 0])
            else:
                lo = 1
                while fits(lo * 2):
                    lo *= 2
                hi = lo * 2  # bisection on the first scale that does not fit
                while hi - lo > 1:
                    mid = (lo + hi) // 2
                    if fits(mid):
                        lo = mid
                    else:
                        hi = mid
                s = G.make_supercell(base, (lo, lo, lo))
                r = run(s, p0)
                rows.append([budget_bytes, lo, r.atoms, estimate_bytes(s, params, p0), "ok", r.time_s])
        elif mode == "density":
            header = "density_factor,atoms,edges,time_s"
            for f in densities:
                sc = (1.0 / f) ** (1.0 / 3.0)
                s = G.AtomicSystem(base.positions * sc, base.lattice * sc, base.species, base.pbc)
                r = run(s, setup.partitions[0])
                rows.append([float(f), r.atoms, r.edges, r.time_s])
        else:
            cols = ["_".join(c.lower().split()) + "_s" for c in G.StepTiming.category_names()]
            header = ",".join(["p", "atoms"] + cols + ["total_s"])
            for p in setup.partitions:
                r = run(base, p)
                m = r.mean
                rows.append([p, r.atoms, m.graph_creation, m.feature_calculation, m.forward_pass,
                             m.backward_pass, m.total()])
        text = io.StringIO()
        text.write(header + "\n")
        for row in rows:
            text.write(",".join(_csv_num(x) for x in row) + "\n")
        if out_path:
            try:
                with open(out_path, "w") as f:
                    f.write(text.getvalue())
            except OSError:
                raise G.Error(f"cannot write file: {out_path}")
        else:
            out.write(text.getvalue())
        return EXIT_OK
    except Exception as e:
        print(f"runtime error: {e}", file=err)
        return EXIT_RUNTIME


def md(setup: Setup, steps: int, dt: float = 1.0, temperature: float = 300.0, out_path: str = "",
       timing_path: str = "", traj_prefix: str = "", snapshot_every: int = 0, paired: bool = False,
       pair_tol: float = 1e-6, out=sys.stdout, err=sys.stderr) -> int:
    """graphmd_cli.cpp:299-355: NVE run on the GPU (the whole trajectory stays
    on the device); --paired reruns with one partition and compares the
    final positions."""
    try:
        system, params = setup.system(), setup.params()
        if dt < 0.0:
            raise G.Error("time step must be >= 0")
        opts = G.MDOptions(dt=dt, steps=steps, partitions=setup.partitions[0], threads=setup.threads,
                           allow_narrow=setup.allow_narrow, seed=setup.seed, init_temperature=temperature,
                           energy_csv=out_path, timing_csv=timing_path, trajectory_xyz=traj_prefix,
                           snapshot_every=snapshot_every)
    except Exception as e:
        print(f"config error: {e}", file=err)
        return EXIT_CONFIG
    try:
        res = G.run_md(system, params, opts, setup.device)
        last, first = res.records[-1], res.records[0]
        print(f"steps={steps} E_total_final={last.total:.9g} "
              f"drift/atom={abs(last.total - first.total) / system.size():.6g}", file=out)
        if paired:
            ser = G.MDOptions(**{**opts.__dict__, "partitions": 1, "energy_csv": "", "timing_csv": "",
                                 "trajectory_xyz": ""})
            ref = G.run_md(system, params, ser, setup.device)
            dmax = float(np.abs(res.state.current_system().positions
                                - ref.state.current_system().positions).max())
            print(f"paired max|dx|={dmax:.6g} (p={opts.partitions} vs serial)", file=out)
            if dmax > pair_tol:
                return EXIT_TOLERANCE
        return EXIT_OK
    except Exception as e:
        print(f"runtime error: {e}", file=err)
        return EXIT_RUNTIME


def _ints(s: str) -> List[int]:
    return [int(x) for x in s.split(",") if x.strip()]


def main(argv: Optional[Sequence[str]] = None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2506_02023_b200.harness",
                                 description="distributed message-passing potential toolkit (B200)")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def common(sp, need_fixture=True):
        sp.add_argument("--fixture", required=need_fixture, default="", help="input extended-XYZ file")
        sp.add_argument("--reps", type=_ints, default=[1, 1, 1], help="supercell repetitions a,b,c")
        sp.add_argument("--partitions", type=_ints, default=[1, 2, 4], help="partition counts")
        sp.add_argument("--threads", type=int, default=0, help="worker threads (accepted, unused)")
        sp.add_argument("--cutoff", type=float, default=4.0, help="atom graph cutoff (A)")
        sp.add_argument("--threebody-cutoff", type=float, default=0.0, help="three-body cutoff (A), 0 disables")
        sp.add_argument("--seed", type=int, default=12345, help="parameter / velocity seed")
        sp.add_argument("--allow-narrow", action="store_true", help="permit slabs narrower than the cutoff")
        sp.add_argument("--device", type=int, default=0)

    a_ = sub.add_parser("audit", help="partitioned vs one-partition tolerance check")
    common(a_)
    a_.add_argument("--tol-energy", type=float, default=2e-5)
    a_.add_argument("--tol-force", type=float, default=2e-4)
    a_.add_argument("--tol-stress", type=float, default=2e-6)
    a_.add_argument("--corrupt-plan", action="store_true", help="fault injection (must fail)")
    b_ = sub.add_parser("bench", help="scaling benchmark CSV emitter")
    common(b_)
    b_.add_argument("--mode", default="strong")
    b_.add_argument("--repeat", type=int, default=20)
    b_.add_argument("--keep-last", type=int, default=10)
    b_.add_argument("--budget-bytes", type=int, default=0)
    b_.add_argument("--densities", type=lambda s: [float(x) for x in s.split(",")], default=[0.5, 1.0, 2.0])
    b_.add_argument("--out", default="")
    m_ = sub.add_parser("md", help="NVE molecular dynamics")
    common(m_)
    m_.add_argument("--steps", type=int, default=100)
    m_.add_argument("--dt", type=float, default=1.0)
    m_.add_argument("--temperature", type=float, default=300.0)
    m_.add_argument("--out", default="")
    m_.add_argument("--timing-out", default="")
    m_.add_argument("--traj", default="")
    m_.add_argument("--snapshot-every", type=int, default=0)
    m_.add_argument("--paired", action="store_true")
    m_.add_argument("--pair-tol", type=float, default=1e-6)
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:  # argparse: bad flags are configuration errors
        return EXIT_CONFIG if e.code else EXIT_OK
    if len(a.reps) != 3:
        print("config error: --reps takes three integers", file=sys.stderr)
        return EXIT_CONFIG
    setup = Setup(a.fixture, a.reps, a.partitions, a.threads, a.cutoff, a.threebody_cutoff, a.seed,
                  a.allow_narrow, a.device)
    if a.cmd == "audit":
        return audit(setup, a.tol_energy, a.tol_force, a.tol_stress, a.corrupt_plan)
    if a.cmd == "bench":
        return bench(setup, a.mode, a.repeat, a.keep_last, a.budget_bytes, a.densities, a.out)
    return md(setup, a.steps, a.dt, a.temperature, a.out, a.timing_out, a.traj, a.snapshot_every,
              a.paired, a.pair_tol)


if __name__ == "__main__":
    sys.exit(main())

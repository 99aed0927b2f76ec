"""The reference's own benchmark harness driving the device planners.

`run_bench` (bench.py:221-309), its CSV schema (bench.py:31) and `fit_scaling`
(bench.py:353-385) are imported from the reference package installed
unmodified under baseline/_ref (`pip install --target baseline/_ref`, see
DESIGN.md); the test skips where that install is absent.  The harness times
bench_plugin's planners exactly as it times its own CPU planners.
"""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

from fcb_testutil import ROOT

pytestmark = pytest.mark.gpu


def _reference_bench():
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "flowcover")):
        pytest.skip("reference not installed under baseline/_ref")
    if path not in sys.path:
        sys.path.insert(0, path)
    import flowcover.bench as rb

    return rb


def test_reference_run_bench_times_b200_planners(tmp_path):
    rb = _reference_bench()
    from paper_2511_11514_b200 import bench_plugin

    spec = rb.BenchSpec(methods=("stein", "sinkhorn"), model="diff_drive",
                        horizons=(100, 200, 300, 400), reps=1, metric_samples=300)
    planners = bench_plugin.b200_planners(spec, rb.PlannerRun, reference_names=True)
    _, metric = rb.standard_planners(spec)  # the reference's coverage metric (CPU)
    csv = tmp_path / "bench.csv"
    recs = rb.run_bench(spec, planners=planners, metric=metric, csv_path=csv)
    assert len(recs) == 8 and all(r.status == "ok" for r in recs), [r.status for r in recs]
    lines = csv.read_text().splitlines()
    assert lines[0] == rb.CSV_HEADER
    parsed = [rb.BenchRecord.from_csv_row(l) for l in lines[1:]]
    assert [(r.method, r.horizon) for r in parsed] == [(r.method, r.horizon) for r in recs]
    for method in ("stein", "sinkhorn"):
        fit = rb.fit_scaling(recs, method, "total")
        assert np.isfinite(fit.alpha) and fit.num_horizons == 4
    # the device planner's coverage at T=100 agrees with the reference's own planner
    ref_planners, _ = rb.standard_planners(spec)
    ref_cov = metric(ref_planners["stein"](100, 1).trajectory)
    ours = next(r for r in recs if r.method == "stein" and r.horizon == 100).coverage
    assert ours == pytest.approx(ref_cov, rel=0.01)

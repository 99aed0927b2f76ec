"""Artifact files (reference io.py:1-141): files the reference wrote read back
bit for bit, and files written here byte-identical to the reference's."""

from __future__ import annotations

import os

import numpy as np
import pytest

import paper_2511_11514_b200 as fc
from fcb_testutil import GOLDEN, load_golden
from paper_2511_11514_b200 import io as fio

IO = os.path.join(GOLDEN, "io")


def _need(name):
    path = os.path.join(IO, name)
    if not os.path.exists(path):
        pytest.skip(f"golden file {name} missing (tests/golden/make_golden_r2.py --only tspio)")
    return path


def test_trajectory_roundtrip_matches_reference_file(tmp_path):
    path = _need("traj_diff_drive.csv")
    m = fc.differential_drive()
    traj = fio.read_trajectory(path, m)
    assert traj.S.shape == (26, 3) and traj.U.shape == (25, 2) and traj.dt == 0.05
    out = tmp_path / "t.csv"
    fio.write_trajectory(out, traj, m)
    assert out.read_bytes() == open(path, "rb").read()


@pytest.mark.parametrize("name,names", [("points_named.csv", ("x", "y", "z")),
                                        ("points_plain.csv", None)])
def test_points_roundtrip_matches_reference_file(tmp_path, name, names):
    path = _need(name)
    P = fio.read_points(path)
    out = tmp_path / "p.csv"
    fio.write_points(out, P, names=names)
    assert out.read_bytes() == open(path, "rb").read()


def test_metrics_roundtrip(tmp_path):
    path = _need("metrics.json")
    payload = fio.read_metrics(path)
    out = tmp_path / "m.json"
    fio.write_metrics(out, payload)
    assert out.read_bytes() == open(path, "rb").read()


def test_format_errors_carry_the_row(tmp_path):
    m = fc.single_integrator_2d()
    bad = tmp_path / "bad.csv"
    bad.write_text(fio.trajectory_header(m) + "\n0.0,0.1,0.1,1.0,1.0\n0.05,0.2,x,,\n")
    with pytest.raises(fio.TrajectoryFormatError) as e:
        fio.read_trajectory(bad, m)
    assert e.value.row == 3
    bad.write_text("t,x\n0.0,0.1,0.1,1.0,1.0\n")
    with pytest.raises(fio.TrajectoryFormatError) as e:
        fio.read_trajectory(bad, m)
    assert e.value.row == 1
    pts = tmp_path / "pts.csv"
    pts.write_text("1.0,2.0\n3.0\n")
    with pytest.raises(fio.TrajectoryFormatError) as e:
        fio.read_points(pts)
    assert e.value.row == 2
    np.testing.assert_array_equal(fio.read_points(_write(tmp_path, "a,b\n\n1.5,2.5\n")), [[1.5, 2.5]])


def _write(tmp_path, text):
    p = tmp_path / "x.csv"
    p.write_text(text)
    return p


def test_resample_arclength_matches_reference():
    """Host half of the baseline's tracking stage (tsp.py:150-167), bit for bit."""
    from paper_2511_11514_b200.tsp import resample_arclength
    g = load_golden("track_cases.npz")
    np.testing.assert_array_equal(resample_arclength(g["rs_in"], 37), g["rs_out"])
    np.testing.assert_array_equal(resample_arclength(g["rs_in"][:2], 5), g["rs_single"])
    np.testing.assert_array_equal(resample_arclength(np.ones((3, 2)), 4), np.ones((4, 2)))
    with pytest.raises(ValueError):
        resample_arclength(np.ones((2, 2)), 0)

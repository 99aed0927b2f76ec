"""The C ABI surface: the library loads and exports every declared symbol.

CPU-only: nothing here launches a kernel.
"""

from __future__ import annotations

import ctypes
import os
import re
import subprocess

from fcb_testutil import ROOT

HEADER = os.path.join(ROOT, "include", "flowcover_b200.h")
LIB = os.path.join(ROOT, "paper_2511_11514_b200", "libflowcover_b200.so")


def declared_symbols() -> list[str]:
    text = open(HEADER).read()
    return sorted(set(re.findall(r"FCB_API\s+[\w\s\*]+?\b(fcb_\w+)\s*\(", text)))


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for name in ("fcb_ot_solve", "fcb_sinkhorn_flow", "fcb_sinkhorn_divergence", "fcb_gmm_eval",
                 "fcb_median_bandwidth", "fcb_stein_flow", "fcb_rollout", "fcb_lqr_solve",
                 "fcb_plan_update"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True)
    exported = set(re.findall(r"\bT (fcb_\w+)", out.stdout))
    assert set(declared_symbols()) <= exported


def test_python_binding_matches_header():
    from paper_2511_11514_b200 import _lib

    assert set(_lib.SIGNATURES) == set(declared_symbols())
    lib = _lib.load()
    assert lib.fcb_version().decode().startswith("flowcover-b200")
    assert _lib.launch_count() >= 0


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True)
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches

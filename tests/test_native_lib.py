"""The C-ABI library builds for sm_100a, loads, and exports every symbol the
public header declares (no compute call: this runs without a GPU)."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "kifmm_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^int\s+(kifmm_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("kifmm_p2p_blocked_f32", "kifmm_p2p_blocked_f64", "kifmm_hadamard_m2l_c64",
                 "kifmm_hadamard_m2l_c128", "kifmm_laplace_potentials_f32",
                 "kifmm_laplace_matrix_f64", "kifmm_m2l_sweep_f32", "kifmm_fft_forward_f64",
                 "kifmm_leaf_pass_f32"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_2408_07436_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        pytest.fail("libkifmm_b200.so not built: run __graft_entry__.build()")
    lib = ctypes.CDLL(_native.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    # the Python binding declares exactly the header's entry points
    assert sorted(_native.SIGNATURES) == declared_symbols()
    assert lib.kifmm_sm_target() == 100


def test_library_is_sm100a_code():
    from paper_2408_07436_b200 import _native
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    import numpy as np
    from paper_2408_07436_b200 import FmmConfig, hotloops, setup
    pts = np.random.default_rng(0).random((500, 3))
    inst = setup(pts, pts, FmmConfig(depth=2, order_equiv=3))
    with pytest.raises(RuntimeError, match="CUDA"):
        inst.evaluate(np.ones(500))
    with pytest.raises(RuntimeError, match="CUDA"):
        hotloops.laplace_potentials(pts[:, 0], pts[:, 1], pts[:, 2], pts[:, 0], pts[:, 1],
                                    pts[:, 2], np.ones((500, 1)), np.zeros((500, 1)))

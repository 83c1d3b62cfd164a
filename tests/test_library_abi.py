"""CPU-side checks of the C ABI boundary: the in-tree libsknr_b200.so exists,
loads, and exports every function declared in include/sknr_gpu.h; without a
GPU every compute call fails loudly (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sknr_gpu.h")
LIB = os.path.join(ROOT, "paper_2506_14780_b200", "libsknr_b200.so")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sknr_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_reference_surface():
    names = declared_functions()
    for required in ["sknr_problem_create_dense", "sknr_problem_create_points", "sknr_ctransform_of_f",
                     "sknr_ctransform_of_g", "sknr_plan_marginals", "sknr_coupling",
                     "sknr_semi_dual_value", "sknr_restricted_derivatives", "sknr_top_modes",
                     "sknr_solve", "sknr_anneal", "sknr_apply_sym_block", "sknr_apply_sym_t_block"]:
        assert required in names


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "build with __graft_entry__.build()"
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (sknr_[a-z_0-9]+)", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing


def test_library_loads_and_reports_version():
    lib = ctypes.CDLL(LIB)
    buf = ctypes.create_string_buffer(256)
    lib.sknr_version.argtypes = [ctypes.c_char_p, ctypes.c_int]
    assert lib.sknr_version(buf, 256) == 0
    assert buf.value.startswith(b"sknr_b200")


def test_kernels_are_sm100a_sass():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_means_loud_failure():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2506_14780_b200 as sk

    with pytest.raises(RuntimeError, match="no CUDA device"):
        sk.Problem(np.zeros((2, 2)), [0.5, 0.5], [0.5, 0.5], 1.0)


def test_invalid_arguments_mirror_reference_messages():
    import paper_2506_14780_b200 as sk

    with pytest.raises(ValueError, match="weights must sum to 1"):
        sk.Problem(np.zeros((2, 2)), [0.5, 0.6], [0.5, 0.5], 1.0)
    with pytest.raises(ValueError, match="strictly positive"):
        sk.Problem(np.zeros((2, 2)), [1.0, 0.0], [0.5, 0.5], 1.0)
    with pytest.raises(ValueError, match="epsilon must be positive"):
        sk.Problem(np.zeros((2, 2)), [0.5, 0.5], [0.5, 0.5], 0.0)
    with pytest.raises(ValueError, match="measure sizes"):
        sk.Problem(np.zeros((2, 3)), [0.5, 0.5], [0.5, 0.5], 1.0)

"""CPU checks of the C-ABI boundary: libsysml.so builds for sm_100a, loads, and exports
every symbol include/sysml.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "sysml.h")).read()
    return sorted(set(re.findall(r"^SYSML_API\s+[\w\s\*]+?\b(sysml_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_north_star_entry_points():
    syms = header_symbols()
    for name in ("sysml_conv2d", "sysml_conv2d_bwd_filter", "sysml_conv2d_bwd_data", "sysml_bias_add",
                 "sysml_relu_maxpool", "sysml_maxpool_bwd", "sysml_lenet_step", "sysml_sgd_update"):
        assert name in syms


def test_library_builds_and_exports_every_header_symbol():
    from paper_1802_04647_b200 import _build, EXPORTS
    so = _build.build()
    lib = ctypes.CDLL(so)
    syms = header_symbols()
    assert set(syms) == set(EXPORTS), set(syms) ^ set(EXPORTS)
    for name in syms:
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (sysml_\w+)", out))
    assert set(syms) <= exported


def test_library_is_sm100a_and_uses_tcgen05():
    from paper_1802_04647_b200 import _build
    so = _build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_oracle_shares_no_code_with_product():
    # the product never imports/links the oracle and vice versa
    pkg = os.path.join(ROOT, "paper_1802_04647_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", txt).lower(), fn
    osrc = open(os.path.join(ROOT, "oracle", "oracle.c")).read()
    assert "#include \"" not in osrc and "sysml.h" not in osrc.replace("libsysml", "")


def test_binding_fails_loudly_without_cuda():
    import torch
    import paper_1802_04647_b200 as s
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    d = s.conv_desc(1, 1, 4, 4, 1, 3, 3, pad=1, math="fp32")
    with pytest.raises((TypeError, RuntimeError)):
        s.sysml_conv2d(torch.zeros(1, 16), torch.zeros(1, 9), d)

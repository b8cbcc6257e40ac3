"""The C-ABI library builds for sm_100a, loads without a GPU and exports every
entry point include/l0cert_b200.h declares (no compute calls here)."""

import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "l0cert_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(l0_[a-z0-9_]+)\s*\(", text)) - {"l0_trace_cb"})


@pytest.fixture(scope="module")
def lib_path():
    from paper_2502_09502_b200 import build
    return build.build()


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("l0_fista_solve", "l0_prox", "l0_g_value", "l0_g_conjugate",
                 "l0_safe_lower_bound", "l0_power_iteration", "l0_loss_value",
                 "l0_loss_conjugate", "l0_problem_create", "l0_problem_set_comm"):
        assert must in names


def test_library_exports_every_declared_symbol(lib_path):
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (l0_[a-z0-9_]+)\b", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing


def test_ctypes_binding_covers_the_header(lib_path):
    from paper_2502_09502_b200 import native
    lib = native.load_library(lib_path)      # dlopen only: no CUDA context
    assert lib.l0_abi_version() == 1
    assert set(native.EXPORTED) == set(declared_functions())


def test_cubin_is_sm100a(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True)
    assert out.returncode == 0
    assert "sm_100a" in out.stdout

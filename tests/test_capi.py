"""C-ABI library checks that need no GPU: it builds, loads, and exports every
entry point include/gpulsm.h declares; no compute is called."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_1707_05354_b200 as pkg
from paper_1707_05354_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gpulsm.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(lsm_[a-z_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    B.build()
    return pkg.load_library()


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for name in ["lsm_create", "lsm_insert", "lsm_delete", "lsm_update", "lsm_lookup",
                 "lsm_count", "lsm_range", "lsm_cleanup"]:
        assert name in syms


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.check_output(["nm", "-D", "--defined-only", B.LIB]).decode()
    exported = set(line.split()[-1] for line in out.splitlines() if " T " in line)
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    # and the binding declares exactly those signatures
    assert sorted(pkg.SIGNATURES) == declared_symbols()


def test_library_is_sm100a(lib):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", B.LIB]).decode()
    assert "sm_100a" in out


def test_status_strings(lib):
    assert pkg.status_string(0) == "ok"
    assert "batch size" in pkg.status_string(2)


def test_create_argument_checks_without_device(lib):
    h = ctypes.c_void_p()
    assert lib.lsm_create(0, ctypes.byref(h)) == 1          # b == 0
    assert lib.lsm_create(4, None) == 1                     # out NULL
    assert lib.lsm_num_batches(None, None) == 1
    assert lib.lsm_update(None, None, None, None, 4, None) == 1


def test_no_torch_types_in_header():
    txt = open(HEADER).read()
    assert "torch" not in txt.lower().replace("pytorch", "") or "at::" not in txt
    assert "at::Tensor" not in txt and "c10" not in txt

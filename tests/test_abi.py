"""CPU checks of the boundary: libgeig.so builds for sm_100a, loads, exports
every function include/geig.h declares, and fails loudly (no CPU fallback)
when no GPU is present."""
import ctypes
import os
import re
import subprocess

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2206_04993_b200 import build
    return build.build()


def _declared():
    src = open(os.path.join(ROOT, "include", "geig.h")).read()
    return sorted(set(re.findall(r"\b(geig_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for n in ["geig_create", "geig_destroy", "geig_products_cca", "geig_products_dense", "geig_update",
              "geig_step_cca", "geig_step_dense", "geig_run_cca", "geig_get", "geig_init_state",
              "geig_step_cca_host"]:
        assert n in names


def test_library_exports_every_declared_symbol(lib_path):
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (geig_[a-z_0-9]+)", out))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(lib_path)
    for n in _declared():
        assert hasattr(lib, n)


def test_binding_mirrors_the_c_names(lib_path):
    from paper_2206_04993_b200 import geig
    for n in _declared():
        assert hasattr(geig, n), n
    assert set(geig.EXPORTED) == set(_declared())


def test_sm100a_code_in_library(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_no_gpu_fails_loudly(lib_path):
    from paper_2206_04993_b200 import geig
    with pytest.raises(geig.GeigError):
        geig.geig_create(geig.GEIG_CCA, 8, 8, 2, geig.GEIG_MATH_F32, geig.GEIG_DATA_F32, 0.1, 16, 0)


def test_default_build_reads_no_environment():
    """No environment variable changes the library's schedule or numerics:
    getenv appears only inside common.cuh's dev_knob, compiled in only with
    -DGEIG_DEV_KNOBS=1 (developer A/B builds)."""
    csrc = os.path.join(ROOT, "paper_2206_04993_b200", "csrc")
    hits = []
    for f in sorted(os.listdir(csrc)):
        for i, line in enumerate(open(os.path.join(csrc, f)), 1):
            if "getenv" in line:
                hits.append((f, i, line.strip()))
    assert [(f, t) for f, _, t in hits] == [("common.cuh", "return std::getenv(name);")], hits
    src = open(os.path.join(csrc, "common.cuh")).read()
    assert "#if GEIG_DEV_KNOBS\n  return std::getenv(name);" in src

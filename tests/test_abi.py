"""The C-ABI library builds for sm_100a, loads, and exports every symbol include/delimit.h declares.

CPU-only: no compute entry is exercised with real buffers here; on a machine
without an sm_100a device they must refuse (DL_ENODEVICE) rather than fall back.
"""

import ctypes
import os
import re
import subprocess

import pytest
import torch

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "delimit.h")


@pytest.fixture(scope="module")
def lib():
    from paper_1808_01517_b200._build import build_library
    from paper_1808_01517_b200 import _lib

    build_library()
    return _lib.load()


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(dl_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_abi():
    names = declared_symbols()
    assert "dl_chan_contract_f32" in names and "dl_chain_bwd_f32" in names
    assert len(names) >= 11


def test_every_declared_symbol_exported(lib):
    from paper_1808_01517_b200._lib import LIB_PATH, SIGNATURES

    out = subprocess.run(["nm", "-D", "--defined-only", LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b(dl_[a-z0-9_]+)\b", out))
    for name in declared_symbols():
        assert name in exported, name
        assert hasattr(lib, name)
    assert set(SIGNATURES) == set(declared_symbols())


def test_library_is_sm100a_only():
    from paper_1808_01517_b200._lib import LIB_PATH

    res = subprocess.run(["cuobjdump", "--list-elf", LIB_PATH], capture_output=True, text=True)
    archs = set(re.findall(r"sm_\d+a?", res.stdout))
    assert archs == {"sm_100a"}, archs


def test_abi_version_and_workspace_queries(lib):
    assert lib.dl_abi_version() == 105
    n = (3 * 45) * (3 * 45 + 1)
    assert lib.dl_lsc_wgrad_workspace_bytes(3, 3, 45, 45) >= n * 8
    ws = lib.dl_chain_workspace_bytes(1, 3, 3, 90, 45, 45, 90, 1000)
    assert ws >= 3 * 135 * 1000 * 4


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device refusal path")
def test_compute_entries_refuse_without_device(lib):
    from paper_1808_01517_b200._lib import last_error

    st = lib.dl_chan_contract_f32(None, None, None, None, 1, 1, 4, 4, 16, 64, 64, 0, None)
    assert st == 3  # DL_ENODEVICE
    assert last_error()
    assert lib.dl_device_supported() == 0


def test_ops_refuse_cpu_tensors():
    import numpy as np

    import paper_1808_01517_b200 as dl
    from paper_1808_01517_b200.directions import unit_sphere_directions

    s2sh = dl.Signal2SH(4, unit_sphere_directions(30))
    with pytest.raises(dl.DeviceError, match="no CPU path"):
        s2sh(torch.ones(1, 30, 2, 2, 2))
    with pytest.raises(dl.ShapeError):
        s2sh(torch.ones(30, 2, 2, 2))
    with pytest.raises(dl.ShapeError, match="multiple of N"):
        s2sh(torch.ones(1, 29, 2, 2, 2))
    del np

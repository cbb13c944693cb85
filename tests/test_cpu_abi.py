"""The C-ABI library loads and exports every symbol its headers declare (no
GPU needed: only symbol resolution and the pure-host entry points run)."""
import ctypes as C
import os
import re

import pytest

from paper_2411_17651_b200 import abi

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    text = open(os.path.join(REPO, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(psgh?_[a-z_]+)\s*\(", text)))


@pytest.mark.parametrize("header", ["psg.h", "psg_host.h"])
def test_library_exports_every_declared_symbol(header):
    lib = abi.load_library()
    names = declared(header)
    assert names, header
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_version_and_struct_sizes():
    lib = abi.load_library()
    assert b"sm_100a" in lib.psg_version()
    assert abi.ENTRY_DTYPE.itemsize == 176
    assert abi.METRICS_DTYPE.itemsize == 40       # == plansim::RequestMetrics
    assert abi.RANK_KEY_DTYPE.itemsize == 48


def test_context_create_fails_cleanly_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    lib = abi.load_library()
    h = C.c_void_p()
    rc = lib.psg_context_create(0, C.byref(h))
    assert rc in (abi.PSG_ERR_CUDA, abi.PSG_ERR_USAGE)
    assert not h.value


def test_engine_refuses_without_library(tmp_path):
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        abi._lib_backup = abi._lib
        try:
            abi._lib = None
            abi.load_library(str(tmp_path / "missing.so"))
        finally:
            abi._lib = abi._lib_backup


def test_config_struct_matches_the_header():
    """psg_config's C layout (include/psg.h) as ctypes sees it: the SLO fields
    close the struct after emit_iterations."""
    names = [f[0] for f in abi.ConfigC._fields_]
    assert names[-3:] == ["emit_iterations", "ttft_slo", "slo_quantile"]
    assert C.sizeof(abi.ConfigC) == 96

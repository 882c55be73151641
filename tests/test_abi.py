"""The C-ABI library loads, exports every entry point include/gshare_b200.h
declares, and the product path fails loudly (no CPU fallback) without a GPU."""
import ctypes
import os
import re

import pytest

from paper_2309_00558_b200 import backend, build as cuda_build, compiler as cc, engine, workloads as wl
from paper_2309_00558_b200.errors import BackendUnavailableError
from paper_2309_00558_b200.scenario import Scenario

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gshare_b200.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|double|void)\s+(gs_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("gs_run_batch", "gs_session_create", "gs_session_run", "gs_session_download",
                 "gs_session_destroy", "gs_abi_version"):
        assert must in names


def test_library_exports_every_declared_symbol():
    cuda_build.build()
    lib = ctypes.CDLL(backend.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert backend.lib().gs_abi_version() == 2


def test_numpy_structs_match_the_header():
    import oracle
    for name, size in cc.STRUCT_SIZES.items():
        assert oracle.sizeof(name) == size, name


def test_product_path_has_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    sc = Scenario.from_dict(wl.c3(0, windows=3))
    with pytest.raises(BackendUnavailableError):
        engine.run(sc)

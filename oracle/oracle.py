"""ctypes front end of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU legs;
the product package never imports this module.  The oracle consumes the same
compiled batch as the CUDA library and fills the same output records, so a
parity check is a byte comparison of two output dicts.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libgs_oracle.so")

_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or (
            os.path.getmtime(LIB) < os.path.getmtime(os.path.join(HERE, "gs_oracle.c"))):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        _lib = C.CDLL(LIB)
        _lib.gs_oracle_run_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
        _lib.gs_oracle_run_batch.restype = C.c_int
        _lib.gs_oracle_sizeof.argtypes = [C.c_char_p]
        _lib.gs_oracle_sizeof.restype = C.c_int
    return _lib


def run_batch(batch, n_threads: int = 1, rows: bool = True) -> dict:
    """Simulate every run of ``batch`` on the CPU; returns the output arrays."""
    from paper_2309_00558_b200.abi import make_batch_struct, make_out_struct
    out = batch.alloc_outputs(rows=rows)
    b = make_batch_struct(batch)
    o = make_out_struct(out)
    lib().gs_oracle_run_batch(C.byref(b), C.byref(o), int(n_threads))
    return out


def sizeof(name: str) -> int:
    return lib().gs_oracle_sizeof(name.encode())

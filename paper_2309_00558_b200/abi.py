"""ctypes view of include/gshare_b200.h.

Builds ``gs_batch_t`` / ``gs_out_t`` from the numpy arrays of a compiled
``Batch`` without copying; the arrays must stay alive for the call.
"""
from __future__ import annotations

import ctypes as C

import numpy as np


class GsBatch(C.Structure):
    _fields_ = [
        ("n_runs", C.c_int32), ("n_funcs", C.c_int32), ("n_points", C.c_int32),
        ("n_inits", C.c_int32), ("n_counts", C.c_int64), ("n_names", C.c_int64),
        ("n_fn_rows", C.c_int64), ("n_gpu_rows", C.c_int64), ("n_glob_rows", C.c_int64),
        ("n_placements", C.c_int64), ("n_id_splits", C.c_int64),
        ("runs", C.c_void_p), ("funcs", C.c_void_p), ("points", C.c_void_p),
        ("inits", C.c_void_p), ("counts", C.c_void_p), ("names", C.c_void_p),
        ("id_splits", C.c_void_p),
    ]


class GsOut(C.Structure):
    _fields_ = [("fn_rows", C.c_void_p), ("gpu_rows", C.c_void_p), ("glob_rows", C.c_void_p),
                ("placements", C.c_void_p), ("status", C.c_void_p), ("summary", C.c_void_p)]


def _ptr(a):
    if a is None:
        return None
    assert isinstance(a, np.ndarray) and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def make_batch_struct(batch) -> GsBatch:
    b = GsBatch()
    b.n_runs = len(batch)
    b.n_funcs = len(batch.funcs)
    b.n_points = len(batch.points)
    b.n_inits = batch.n_inits
    b.n_counts = len(batch.counts)
    b.n_names = len(batch.names)
    b.n_fn_rows = batch.n_fn_rows
    b.n_gpu_rows = batch.n_gpu_rows
    b.n_glob_rows = batch.n_glob_rows
    b.n_placements = batch.n_placements
    b.runs = _ptr(batch.runs)
    b.funcs = _ptr(batch.funcs)
    b.points = _ptr(batch.points)
    b.inits = _ptr(batch.inits)
    b.counts = _ptr(batch.counts)
    b.names = _ptr(batch.names)
    b.n_id_splits = len(batch.id_splits)
    b.id_splits = _ptr(batch.id_splits) if len(batch.id_splits) else None
    return b


def make_out_struct(out: dict) -> GsOut:
    o = GsOut()
    for name in ("fn_rows", "gpu_rows", "glob_rows", "placements", "status", "summary"):
        setattr(o, name, _ptr(out.get(name)))
    return o

"""ctypes binding of liblbfs.so (include/lbfs.h).

The library is the product: there is no Python or CPU fallback for anything
it does. A missing library or a missing GPU raises immediately.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "_native" / "liblbfs.so"

LBFS_OK = 0
LBFS_EINVAL = -1
LBFS_ECUDA = -2
LBFS_ENCCL = -3
LBFS_ENOMEM = -4

_i64 = ctypes.c_int64
_p = ctypes.c_void_p
_lock = threading.Lock()
_lib = None


class Layer(ctypes.Structure):
    _fields_ = [("input", _i64), ("edges", _i64), ("discovered", _i64)]


class Timing(ctypes.Structure):
    _fields_ = [("bfs_ms", ctypes.c_double), ("init_ms", ctypes.c_double),
                ("expand_ms", ctypes.c_double), ("cluster_ms", ctypes.c_double),
                ("finalize_ms", ctypes.c_double), ("d2h_ms", ctypes.c_double),
                ("levels", _i64), ("kernel_launches", _i64), ("edges", _i64), ("reached", _i64)]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class DeviceInfo(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("sm_count", ctypes.c_int), ("cc_major", ctypes.c_int),
                ("cc_minor", ctypes.c_int), ("l2_bytes", _i64), ("hbm_bytes", _i64),
                ("smem_per_block_optin", _i64), ("name", ctypes.c_char * 256)]


# name -> (restype, argtypes); every symbol include/lbfs.h declares.
SIGNATURES = {
    "lbfs_last_error": (ctypes.c_char_p, []),
    "lbfs_device_info_get": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(DeviceInfo)]),
    "lbfs_kernel_launch_count": (_i64, []),
    "lbfs_host_alloc": (ctypes.c_int, [_i64, ctypes.POINTER(_p)]),
    "lbfs_host_free": (None, [_p]),
    "lbfs_rmat_edges": (ctypes.c_int, [ctypes.c_int, _i64, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_double, _p, _p, _p]),
    "lbfs_permute_edges": (ctypes.c_int, [_i64, ctypes.c_uint64, _p, _p, _i64]),
    "lbfs_csr_build": (ctypes.c_int, [_i64, _p, _p, _i64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_p)]),
    "lbfs_csr_build_rmat": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                           ctypes.c_double, _p, ctypes.c_int, ctypes.c_uint64,
                                           ctypes.POINTER(_p)]),
    "lbfs_csr_build_lattice": (ctypes.c_int, [_i64, _i64, ctypes.c_int, ctypes.c_uint64, ctypes.POINTER(_p)]),
    "lbfs_csr_info": (ctypes.c_int, [_p, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "lbfs_csr_download": (ctypes.c_int, [_p, _p, _p]),
    "lbfs_csr_destroy": (None, [_p]),
    "lbfs_graph_create": (ctypes.c_int, [_i64, _p, _p, _i64, ctypes.c_int, ctypes.POINTER(_p)]),
    "lbfs_graph_create_from_csr": (ctypes.c_int, [_p, ctypes.c_int, ctypes.POINTER(_p)]),
    "lbfs_graph_create_partitioned": (ctypes.c_int, [_p, ctypes.c_int, _p, ctypes.POINTER(_p)]),
    "lbfs_graph_gpus": (ctypes.c_int, [_p, ctypes.POINTER(ctypes.c_int)]),
    "lbfs_graph_destroy": (None, [_p]),
    "lbfs_graph_info": (ctypes.c_int, [_p, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "lbfs_bfs": (ctypes.c_int, [_p, _i64, ctypes.c_int, _p, _p, ctypes.POINTER(Layer), _i64,
                                ctypes.POINTER(_i64), ctypes.POINTER(Timing)]),
    "lbfs_bfs_device": (ctypes.c_int, [_p, _i64, ctypes.c_int, _p, _p, ctypes.POINTER(Layer), _i64,
                                       ctypes.POINTER(_i64), ctypes.POINTER(Timing)]),
    "lbfs_graph_last_layers": (ctypes.c_int, [_p, ctypes.POINTER(Layer), _i64, ctypes.POINTER(_i64)]),
    "lbfs_graph_last_levels": (ctypes.c_int, [_p, _p]),
    "lbfs_set_device": (ctypes.c_int, [ctypes.c_int]),
    "lbfs_validate_tree": (ctypes.c_int, [_p, _i64, _p, _p]),
    "lbfs_validate_tree_device": (ctypes.c_int, [_p, _i64, _p, _p]),
    "lbfs_part_create": (ctypes.c_int, [_i64, _p, _p, _i64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_p)]),
    "lbfs_part_create_from_csr": (ctypes.c_int, [_p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_p)]),
    "lbfs_part_info": (ctypes.c_int, [_p, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                      ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "lbfs_part_start": (ctypes.c_int, [_p, _i64, _p, _p]),
    "lbfs_part_expand": (ctypes.c_int, [_p, _p]),
    "lbfs_part_pack": (ctypes.c_int, [_p, _p, _p]),
    "lbfs_part_merge": (ctypes.c_int, [_p, _p, _p, _p]),
    "lbfs_part_sync": (ctypes.c_int, [_p, _p, _p]),
    "lbfs_part_level_done": (ctypes.c_int, [_p, _p, ctypes.POINTER(Layer), ctypes.POINTER(ctypes.c_int)]),
    "lbfs_part_finish": (ctypes.c_int, [_p, _p, _p, _p]),
    "lbfs_part_resolve_count": (ctypes.c_int, [_p, ctypes.POINTER(_i64)]),
    "lbfs_part_plan": (ctypes.c_int, [_p, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "lbfs_nccl_unique_id": (ctypes.c_int, [_p]),
    "lbfs_part_attach_nccl": (ctypes.c_int, [_p, _p, ctypes.c_int, ctypes.c_int]),
    "lbfs_part_bfs": (ctypes.c_int, [_p, _i64, _p, _p, ctypes.c_int, ctypes.POINTER(Layer), _i64,
                                     ctypes.POINTER(_i64), ctypes.POINTER(Timing)]),
}


def load(path: Path | str | None = None):
    """Load liblbfs.so (no GPU needed to load; calls need one)."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path else Path(os.environ.get("LBFS_LIB") or LIB_PATH)
        if not p.exists():
            raise RuntimeError(f"{p} is not built: run `python -c 'import __graft_entry__ as g; g.build()'`"
                               " (there is no CPU fallback)")
        lib = ctypes.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def last_error() -> str:
    return load().lbfs_last_error().decode(errors="replace")


def check(rc: int) -> None:
    """Map an LBFS_E* code to the reference's exception types."""
    if rc == LBFS_OK:
        return
    msg = last_error()
    if rc == LBFS_EINVAL:
        raise AssertionError(msg)
    if rc == LBFS_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"liblbfs error {rc}: {msg}")


def ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def device_info(device: int = 0) -> DeviceInfo:
    info = DeviceInfo()
    check(load().lbfs_device_info_get(device, ctypes.byref(info)))
    return info


def kernel_launch_count() -> int:
    return int(load().lbfs_kernel_launch_count())


# ---------------------------------------------------------------- pinned pool
_pool: dict[int, list[int]] = {}
_pool_lock = threading.Lock()
_POOL_KEEP = 4  # free buffers kept per size


def _pool_put(nbytes: int, addr: int) -> None:
    with _pool_lock:
        lst = _pool.setdefault(nbytes, [])
        if len(lst) < _POOL_KEEP:
            lst.append(addr)
            return
    load().lbfs_host_free(addr)


def pinned_empty(count: int, dtype=np.int32) -> np.ndarray:
    """numpy array backed by page-locked memory from a small pool; the buffer
    returns to the pool when the array (and its views) are garbage."""
    import weakref

    dt = np.dtype(dtype)
    nbytes = max(int(count) * dt.itemsize, 16)
    with _pool_lock:
        lst = _pool.get(nbytes)
        addr = lst.pop() if lst else None
    if addr is None:
        out = ctypes.c_void_p()
        check(load().lbfs_host_alloc(nbytes, ctypes.byref(out)))
        addr = out.value
    raw = (ctypes.c_byte * nbytes).from_address(addr)
    weakref.finalize(raw, _pool_put, nbytes, addr)
    return np.frombuffer(raw, dtype=dt, count=int(count))

"""Build and load the native library (``_lib/liblscan.so``) — the C ABI of
``include/lscan.h`` — through ctypes.

There is no fallback: if the library is missing, was built for another
architecture, or no CUDA device is visible, every device entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from typing import List, Optional

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
CSRC = os.path.join(PKG_DIR, "csrc")
INCLUDE = os.path.join(REPO_DIR, "include")
LIB_DIR = os.path.join(PKG_DIR, "_lib")
LIB_PATH = os.path.join(LIB_DIR, "liblscan.so")

SOURCES = ["lscan_api.cu", "lscan_host.cu", "lscan_inst_i32.cu", "lscan_inst_i64.cu",
           "lscan_inst_f32.cu", "lscan_inst_f64.cu"]
HEADERS = ["lscan_common.cuh", "lscan_ptx.cuh", "lscan_cluster.cuh", "lscan_generic.cuh", "lscan_scan_ws2.cuh", "lscan_ordered.cuh", "lscan_dispatch.h",
           "lscan_inst.cuh"]
ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]

# ls_status (include/lscan.h)
LS_OK = 0
LS_ERR_INVALID_ARG = 1
LS_ERR_UNSUPPORTED_DTYPE = 2
LS_ERR_CUDA = 3
LS_ERR_LIVENESS = 4
LS_ERR_PROTOCOL = 5
LS_ERR_WORKSPACE = 6

# ls_dtype
LS_I32, LS_I64, LS_F32, LS_F64 = 0, 1, 2, 3

# ls_op
LS_OP_ADD, LS_OP_MAX, LS_OP_MIN = 0, 1, 2

# ls_scan_host_ex flags
LS_HOST_EXCLUSIVE, LS_HOST_ORDERED = 1, 2
OPS = {"add": LS_OP_ADD, "max": LS_OP_MAX, "min": LS_OP_MIN}

EXPORTED = [
    "ls_workspace_bytes", "ls_workspace_init", "ls_inclusive_scan", "ls_exclusive_scan", "ls_inclusive_sum",
    "ls_exclusive_sum", "ls_reduce", "ls_reduce_sum", "ls_carry_from_totals", "ls_scan_host",
    "ls_inclusive_sum_host", "ls_debug_config", "ls_debug_perturb",
    "ls_workspace_error", "ls_status_string", "ls_last_error_detail", "ls_abi_version",
    "ls_query_config", "ls_launch_count", "ls_xchg_bytes", "ls_inclusive_scan_multi", "ls_exclusive_scan_multi",
    "ls_device_alloc", "ls_device_free", "ls_ipc_get_handle", "ls_ipc_open", "ls_ipc_close", "ls_debug_slot_stress",
    "ls_debug_force_path", "ls_query_cluster", "ls_query_multi_config", "ls_ordered_scan", "ls_scan_host_ex",
]


def _inputs() -> List[str]:
    return ([os.path.join(CSRC, s) for s in SOURCES + HEADERS]
            + [os.path.join(INCLUDE, "lscan.h")])


def needs_build() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    t = os.path.getmtime(LIB_PATH)
    return any(os.path.getmtime(p) > t for p in _inputs())


def build(force: bool = False, verbose: bool = False, extra: Optional[List[str]] = None) -> str:
    """nvcc the CUDA sources into ``_lib/liblscan.so`` for sm_100a (one
    object per translation unit, compiled in parallel, then linked)."""
    if not force and not needs_build():
        return LIB_PATH
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(LIB_DIR, exist_ok=True)
    objdir = os.path.join(LIB_DIR, "obj")
    os.makedirs(objdir, exist_ok=True)
    nvcc = os.environ.get("NVCC", "nvcc")
    flags = ["-O3", "-std=c++17", *ARCH_FLAGS, "-lineinfo", "-Xcompiler", "-fPIC", f"-I{INCLUDE}"]
    if verbose:
        flags.append("-Xptxas=-v")
    if extra:
        flags += extra

    def compile_one(src):
        obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
        subprocess.run([nvcc, *flags, "-c", "-o", obj, os.path.join(CSRC, src)], check=True)
        return obj

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = LIB_PATH + ".tmp"
    subprocess.run([nvcc, *ARCH_FLAGS, "-shared", "-o", tmp, *objs], check=True)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


_lib = None
_lock = threading.Lock()


def lib():
    """The loaded library; raises if it is absent (no silent fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"native library {LIB_PATH} is missing; run __graft_entry__.build() "
                "(or python -c 'import paper_1604_04815_b200._native as n; n.build()')")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, sz, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_size_t, ctypes.c_int
        sig = {
            "ls_workspace_bytes": (sz, [ci, i64]),
            "ls_workspace_init": (ci, [vp, sz, vp]),
            "ls_inclusive_scan": (ci, [ci, ci, vp, vp, i64, vp, vp, vp, sz, vp]),
            "ls_exclusive_scan": (ci, [ci, ci, vp, vp, i64, vp, vp, vp, sz, vp]),
            "ls_inclusive_sum": (ci, [ci, vp, vp, i64, vp, vp, vp, sz, vp]),
            "ls_exclusive_sum": (ci, [ci, vp, vp, i64, vp, vp, vp, sz, vp]),
            "ls_reduce": (ci, [ci, ci, vp, i64, vp, vp, sz, vp]),
            "ls_reduce_sum": (ci, [ci, vp, i64, vp, vp, sz, vp]),
            "ls_carry_from_totals": (ci, [ci, ci, vp, i64, i64, vp, vp]),
            "ls_scan_host": (ci, [ci, ci, vp, vp, i64, ci, ci]),
            "ls_scan_host_ex": (ci, [ci, ci, vp, vp, i64, ci, ci]),
            "ls_ordered_scan": (ci, [ci, ci, vp, vp, i64, ci, vp, vp, vp]),
            "ls_inclusive_sum_host": (ci, [ci, vp, vp, i64, ci, ci]),
            "ls_debug_config": (ci, [i64, i64, ci]),
            "ls_debug_perturb": (ci, [i64, i64, i64]),
            "ls_workspace_error": (ci, [vp, sz, vp]),
            "ls_status_string": (ctypes.c_char_p, [ci]),
            "ls_last_error_detail": (ctypes.c_char_p, []),
            "ls_abi_version": (ci, []),
            "ls_query_config": (ci, [ci, i64, ctypes.POINTER(ctypes.c_int64)]),
            "ls_launch_count": (i64, []),
            "ls_xchg_bytes": (sz, [ci, ci, i64]),
            "ls_inclusive_scan_multi": (ci, [ci, ci, vp, vp, i64, vp, vp, vp, sz, ci, ci, vp, sz, vp, ci, vp]),
            "ls_exclusive_scan_multi": (ci, [ci, ci, vp, vp, i64, vp, vp, vp, sz, ci, ci, vp, sz, vp, ci, vp]),
            "ls_device_alloc": (ci, [sz, ctypes.POINTER(ctypes.c_void_p)]),
            "ls_device_free": (ci, [vp]),
            "ls_ipc_get_handle": (ci, [vp, vp]),
            "ls_ipc_open": (ci, [vp, ctypes.POINTER(ctypes.c_void_p)]),
            "ls_ipc_close": (ci, [vp]),
            "ls_debug_slot_stress": (ci, [ci, i64, ci, ctypes.POINTER(ctypes.c_int64)]),
            "ls_debug_force_path": (ci, [ci]),
            "ls_query_cluster": (ci, [ci, ctypes.POINTER(ctypes.c_int64)]),  # out[6]
            "ls_query_multi_config": (ci, [ci, i64, ctypes.POINTER(ctypes.c_int64)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.ls_abi_version() != 1:
            raise RuntimeError("liblscan ABI version mismatch")
        _lib = L
        return _lib


def status_string(code: int) -> str:
    return lib().ls_status_string(code).decode()


def last_detail() -> str:
    return (lib().ls_last_error_detail() or b"").decode(errors="replace")


def launch_count() -> int:
    return int(lib().ls_launch_count())

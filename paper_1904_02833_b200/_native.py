"""Loader for the in-tree CUDA library (libsoftsnake_b200.so).

There is no fallback: if the library is missing or CUDA is unavailable the
calls raise, so a silent CPU path can never stand in for the GPU one.
"""
from __future__ import annotations

import ctypes as C
import os

from ._abi import (SsEnvStats, SsLinkMeshOut, SsLinkMeshParams, SsParams, SsStateView,
                   SsSystemView, SsTopology)

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib")
LIB_PATH = os.environ.get("SS_LIB_OVERRIDE") or os.path.join(LIB_DIR, "libsoftsnake_b200.so")

SS_EINVAL, SS_ECUDA, SS_ENOMEM, SS_EUNSUP = -1, -2, -3, -4

_lib = None

# every symbol include/softsnake_b200.h declares, with its ctypes signature
_vp, _dp, _ip, _i = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int32), C.c_int
SIGNATURES = {
    "ss_abi_version": (C.c_int, []),
    "ss_last_error": (C.c_char_p, []),
    "ss_build_id": (C.c_char_p, []),
    "ss_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "ss_create": (C.c_int, [C.POINTER(SsTopology), C.POINTER(SsParams), _i, _i, C.POINTER(_vp)]),
    "ss_destroy": (C.c_int, [_vp]),
    "ss_num_envs": (C.c_int, [_vp]),
    "ss_set_state": (C.c_int, [_vp, _i, _i, C.POINTER(SsStateView)]),
    "ss_get_state": (C.c_int, [_vp, _i, _i, C.POINTER(SsStateView)]),
    "ss_get_state_device": (C.c_int, [_vp, _i, _i, C.POINTER(SsStateView)]),
    "ss_set_state_device": (C.c_int, [_vp, _i, _i, C.POINTER(SsStateView)]),
    "ss_step": (C.c_int, [_vp, _dp, _i, _i]),
    "ss_step_device": (C.c_int, [_vp, _vp, _i, _i]),
    "ss_get_stats": (C.c_int, [_vp, _i, _i, C.POINTER(SsEnvStats)]),
    "ss_export_system": (C.c_int, [_vp, _i, C.POINTER(SsSystemView)]),
    "ss_capture_init": (C.c_int, [_vp, _i]),
    "ss_reset_envs": (C.c_int, [_vp, C.POINTER(C.c_int), _i, C.c_uint64, C.c_double, C.c_double]),
    "ss_get_com": (C.c_int, [_vp, _i, _i, _dp]),
    "ss_observe": (C.c_int, [_vp, _i, _i, _dp]),
    "ss_set_gait": (C.c_int, [_vp, _i, _i, _dp, C.POINTER(C.c_int)]),
    "ss_step_gait": (C.c_int, [_vp, _i, _i]),
    "ss_set_channel_targets": (C.c_int, [_vp, _dp, _i]),
    "ss_get_gait": (C.c_int, [_vp, _i, _i, _dp, C.POINTER(C.c_int)]),
    "ss_synchronize": (C.c_int, [_vp]),
    "ss_stream": (_vp, [_vp]),
    "ss_launches_per_frame": (C.c_int, [_vp]),
    "ss_device_bytes": (C.c_int64, [_vp]),
    "ss_kernel_names": (C.c_int, [C.POINTER(C.c_char_p), _i]),
    "ss_solver_info": (C.c_int, [_vp, C.POINTER(C.c_int)]),
    "ss_check_guards": (C.c_int, [_vp, C.POINTER(C.c_int64)]),
    "ss_cluster_stamps": (C.c_int, [_vp, C.POINTER(C.c_longlong)]),
    "ss_profile_frames": (C.c_int, [_vp, _dp, _i, _i, _dp, C.POINTER(C.c_int)]),
    "ss_link_mesh_counts": (C.c_int, [C.POINTER(SsLinkMeshParams), _ip]),
    "ss_build_link_meshes": (C.c_int, [C.POINTER(SsLinkMeshParams), _i, C.POINTER(SsLinkMeshOut)]),
    "ssk_block_forward": (C.c_int, [_vp, _vp, _i, _i, _i, _vp, _vp, _vp]),
    "ssk_block_transpose": (C.c_int, [_vp, _vp, _i, _i, _i, _vp, _vp, _i, _vp]),
    "ssk_block_rowdiag": (C.c_int, [_vp, _vp, _i, _i, _i, _vp, _vp, _vp]),
    "ssk_minv_apply": (C.c_int, [_vp, _vp, _i, _i, _vp, _vp, _i, _vp]),
    "ssk_ereg_apply": (C.c_int, [_vp, _vp, _vp, _i, _vp]),
    "ssk_dot": (C.c_int, [_vp, _vp, _i, _dp, _vp]),
    "ssk_eval_distance": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _i, _vp]),
    "ssk_eval_tetra": (C.c_int, [_vp, _vp, _vp, _vp, C.c_double, _i, _vp, _vp, _i,
                                 C.POINTER(C.c_int), _vp]),
    "ssk_malloc": (C.c_int, [C.POINTER(_vp), C.c_int64, _i]),
    "ssk_free": (C.c_int, [_vp]),
    "ssk_memcpy": (C.c_int, [_vp, _vp, C.c_int64, _i]),
}


PKG_DIR = os.path.dirname(os.path.abspath(__file__))
# nvcc flags of the library build (part of the build id)
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
              "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
              "-diag-suppress", "177"]
ROOT_DIR = os.path.dirname(PKG_DIR)


def source_files() -> list[str]:
    """The files the library is compiled from (the build id covers them)."""
    csrc = os.path.join(PKG_DIR, "csrc")
    if not os.path.isdir(csrc):
        return []
    return [os.path.join(csrc, f) for f in sorted(os.listdir(csrc))
            if f.endswith((".cu", ".cuh", ".h"))] + \
        [os.path.join(ROOT_DIR, "include", "softsnake_b200.h")]


def source_hash(extra: str | None = None) -> str | None:
    """sha256 over the source files' names and bytes (None without sources)."""
    import hashlib
    files = source_files()
    if not files or not all(os.path.exists(f) for f in files):
        return None
    h = hashlib.sha256()
    for f in files:
        h.update(os.path.basename(f).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    h.update((" ".join(NVCC_FLAGS) if extra is None else extra).encode())
    return h.hexdigest()


def embedded_build_id(path: str = LIB_PATH) -> str | None:
    """The build id stored in a library file, read without loading it."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        return None
    k = data.find(b"ss-build-id:")
    if k < 0:
        return None
    end = data.find(b"\0", k)
    return data[k + 12:end].decode(errors="replace")


def lib():
    """The loaded library; raises RuntimeError if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        want = source_hash()
        got = L.ss_build_id().decode()
        if want is not None and got != want and not os.environ.get("SS_LIB_OVERRIDE"):
            raise RuntimeError(f"{LIB_PATH} was built from other sources (build id {got[:12]}, "
                               f"tree {want[:12]}): rerun __graft_entry__.build()")
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().ss_last_error()
    msg = msg.decode() if msg else f"error {rc}"
    if rc in (SS_EINVAL, SS_EUNSUP):
        raise ValueError(msg)
    raise RuntimeError(msg)

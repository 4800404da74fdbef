"""ctypes binding of libfirecell.so (the C ABI declared in include/firecell.h).

This is the product's only path to the hot kernels.  There is no CPU
fallback: if the shared library is missing or a device op is requested
without a CUDA device, the call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
SO_PATH = os.environ.get("FIRECELL_SO") or os.path.join(HERE, "libfirecell.so")  # override: A/B builds
CU_PATH = os.path.join(HERE, "csrc", "firecell.cu")
HEADER = os.path.join(REPO, "include", "firecell.h")

FC_OK, FC_EINVAL, FC_ECUDA = 0, 1, 2
RNG_SPLITMIX, RNG_PHILOX, RNG_INJECT = 0, 1, 2
RNG_MODES = {"splitmix": RNG_SPLITMIX, "philox": RNG_PHILOX, "inject": RNG_INJECT}
SLOPE_ELEVATION, SLOPE_TENSOR = 0, 1
NPARAM = 8
NCOUNTER = 4
T_NEVER = 0x7FFF

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]

# Every symbol include/firecell.h declares (checked by the CPU test suite).
EXPORTS = ("fc_grid_make", "fc_plane_words", "fc_loss_workspace_bytes", "fc_sched_workspace_bytes",
           "fc_state_init",
           "fc_state_reset",
           "fc_state_unpack", "fc_state_jaccard", "fc_state_export", "fc_state_rebase", "fc_host_device_pointer", "fc_inject", "fc_run", "fc_run_pass", "fc_mark_ghosts", "fc_peer_signal", "fc_stream_wait_geq", "fc_activity_scan",
           "fc_contract", "fc_recompute64", "fc_contract_steps", "fc_loss_grad",
           "fc_loss_dense", "fc_adamw", "fc_uniform_grid", "fc_epoch_seed", "fc_build_fields",
           "fc_landscape_build", "fc_landscape_build_ctas",
           "fc_last_cuda_error", "fc_version", "fc_debug_set_trace")


class FcGrid(C.Structure):
    _fields_ = [("height", C.c_int32), ("width", C.c_int32), ("tiles_y", C.c_int32),
                ("tiles_x", C.c_int32), ("members", C.c_int32)]


class FcLandscape(C.Structure):
    _fields_ = [("env", C.c_void_p), ("slope4", C.c_void_p), ("env64", C.c_void_p),
                ("slope32", C.c_void_p),
                ("slope64", C.c_void_p), ("dir32", C.c_void_p), ("cell_side", C.c_double),
                ("slope_mode", C.c_int32),
                ("slope_sign", C.c_int32), ("factor_source", C.c_int32), ("pad_", C.c_int32)]


class FcPeerHalo(C.Structure):
    _fields_ = [("up", C.c_void_p * 4), ("down", C.c_void_p * 4), ("up_tiles_y", C.c_int32),
                ("down_tiles_y", C.c_int32), ("up_flag", C.c_void_p), ("down_flag", C.c_void_p),
                ("seq", C.c_int32), ("pad_", C.c_int32)]


class FcShard(C.Structure):
    _fields_ = [("row0", C.c_int32), ("ghost_top", C.c_int32), ("ghost_bottom", C.c_int32),
                ("member0", C.c_int32), ("peer", C.c_void_p)]


class FcState(C.Structure):
    _fields_ = [("burn0", C.c_void_p), ("burn1", C.c_void_p), ("burned0", C.c_void_p),
                ("burned1", C.c_void_p),
                ("acc", C.c_void_p), ("t_ign", C.c_void_p), ("jac", C.c_void_p),
                ("flags", C.c_void_p), ("counters", C.c_void_p), ("tile_list", C.c_void_p),
                ("list_count", C.c_void_p), ("tile_fire", C.c_void_p), ("tile_first", C.c_void_p),
                ("live", C.c_void_p), ("sched", C.c_void_p), ("init_burning", C.c_void_p),
                ("max_steps", C.c_int32),
                ("t_base", C.c_int32)]


def build(force: bool = False) -> str:
    """Compile csrc/firecell.cu for sm_100a into the package directory."""
    stale = (not os.path.exists(SO_PATH) or
             os.path.getmtime(SO_PATH) < max(os.path.getmtime(CU_PATH), os.path.getmtime(HEADER)))
    if force or stale:
        cmd = ["nvcc", *NVCC_FLAGS, "-o", SO_PATH + ".tmp", CU_PATH]
        subprocess.run(cmd, check=True)
        os.replace(SO_PATH + ".tmp", SO_PATH)
    return SO_PATH


_lock = threading.Lock()
_lib = None


def lib():
    """Load libfirecell.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(SO_PATH):
            raise RuntimeError(
                f"{SO_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (nvcc, sm_100a). There is no CPU fallback.")
        L = C.CDLL(SO_PATH)
        vp, i32, i64, u64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
        G, LS, ST = C.POINTER(FcGrid), C.POINTER(FcLandscape), C.POINTER(FcState)
        SH = C.POINTER(FcShard)
        sig = {
            "fc_grid_make": (None, [i32, i32, i32, G]),
            "fc_plane_words": (C.c_size_t, [G]),
            "fc_loss_workspace_bytes": (C.c_size_t, [G, i32]),
            "fc_sched_workspace_bytes": (C.c_size_t, [G, i32]),
            "fc_state_init": (C.c_int, [G, ST, vp, i64, i32, vp]),
            "fc_state_reset": (C.c_int, [G, ST, vp, i64, i32, vp]),
            "fc_state_unpack": (C.c_int, [G, ST, i32, vp, vp, vp]),
            "fc_state_jaccard": (C.c_int, [G, ST, i32, vp, i64, vp, vp, vp]),
            "fc_state_export": (C.c_int, [G, ST, i32, vp, vp, vp, vp, vp]),
            "fc_host_device_pointer": (C.c_int, [vp, C.POINTER(vp)]),
            "fc_inject": (C.c_int, [G, ST, vp, i32, i32, i32, vp]),
            "fc_state_rebase": (C.c_int, [G, ST, vp]),
            "fc_run": (C.c_int, [G, LS, ST, vp, vp, i32, vp, i32, i32, vp, i32, i32, vp, SH,
                                 C.POINTER(i32), vp]),
            "fc_run_pass": (C.c_int, [G, LS, ST, vp, vp, i32, i32, i32, vp, i32, vp, SH, i32,
                                      C.POINTER(i32), vp]),
            "fc_mark_ghosts": (C.c_int, [G, ST, SH, i32, vp]),
            "fc_activity_scan": (C.c_int, [G, ST, i32, vp]),
            "fc_stream_wait_geq": (C.c_int, [vp, i32, vp]),
            "fc_peer_signal": (C.c_int, [vp, i32, vp]),
            "fc_contract": (C.c_int, [G, ST, vp, i32, vp, vp, vp]),
            "fc_recompute64": (C.c_int, [G, LS, ST, vp, i32, i32, vp, vp, vp, vp]),
            "fc_contract_steps": (C.c_int, [G, ST, vp, vp, vp, i32, vp, vp, vp]),
            "fc_loss_grad": (C.c_int, [G, ST, vp, i64, vp, i32, vp, vp, vp, vp, vp, vp]),
            "fc_loss_dense": (C.c_int, [i32, i32, vp, vp, vp, vp, vp, vp, vp]),
            "fc_adamw": (C.c_int, [vp, vp, vp, i32, i32, vp, dbl, dbl, dbl, dbl, dbl, i32, vp, vp]),
            "fc_uniform_grid": (C.c_int, [u64, i64, i32, i64, i64, i64, i64, vp, vp]),
            "fc_epoch_seed": (u64, [u64, u64]),
            "fc_build_fields": (C.c_int, [G, LS, vp, vp, i32, vp]),
            "fc_landscape_build": (C.c_int, [i32, i32, vp, vp, vp, vp, vp, i32, dbl, i32, vp, vp,
                                             vp, vp, vp]),
            "fc_landscape_build_ctas": (C.c_int, [i32, i32, vp, vp, vp, vp, vp, i32, dbl, i32, vp,
                                                  vp, vp, vp, i32, vp]),
            "fc_last_cuda_error": (C.c_int, []),
            "fc_version": (C.c_char_p, []),
            "fc_debug_set_trace": (None, [vp]),
        }
        for name, (res, args) in sig.items():
            if name == "fc_debug_set_trace" and not hasattr(L, name):
                continue  # diagnostics symbol, absent from older A/B builds
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int, what: str) -> None:
    if rc == FC_OK:
        return
    if rc == FC_EINVAL:
        raise ValueError(f"{what}: invalid argument (firecell EINVAL)")
    raise RuntimeError(f"{what}: CUDA error {lib().fc_last_cuda_error()}")


def grid(height: int, width: int, members: int = 1) -> FcGrid:
    g = FcGrid()
    lib().fc_grid_make(int(height), int(width), int(members), C.byref(g))
    return g


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("firecell needs a CUDA device (B200, sm_100a); no CPU fallback")
    lib()


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def device_ptr(t) -> int:
    """Device address of a CUDA tensor, or of a pinned host tensor mapped
    into the device address space (fc_host_device_pointer)."""
    if t is None:
        return 0
    if t.is_cuda:
        return int(t.data_ptr())
    if not t.is_pinned():
        raise ValueError("host tensor must be pinned to be written by the device")
    out = C.c_void_p()
    check(lib().fc_host_device_pointer(C.c_void_p(t.data_ptr()), C.byref(out)),
          "fc_host_device_pointer")
    return int(out.value or 0)

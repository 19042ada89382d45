"""ctypes binding of libvpipe.so (include/vpipe.h). The library is REQUIRED:
importing this module fails loudly when it is missing — there is no Python
or CPU fallback for any entry point."""

from __future__ import annotations

import ctypes
import os

from .errors import ConfigError, InfeasibleError

_HERE = os.path.dirname(os.path.abspath(__file__))
# VP_LIB_PATH: load an alternative build (e.g. an instrumented one) instead
LIB_PATH = os.environ.get("VP_LIB_PATH") or os.path.join(_HERE, "libvpipe.so")

VP_OK = 0
VP_ERR_ARGS = -1
VP_ERR_INFEASIBLE = -2
VP_ERR_DEADLOCK = -3
VP_ERR_NOMEM = -4
VP_ERR_CAPACITY = -5
VP_ERR_UNSUPPORTED = -6
VP_ERR_NOTIMPL = -7


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libvpipe.so not built at {LIB_PATH}; run `python __graft_entry__.py` (or `python paper_2111_04007_b200/build.py`) "
            "(there is no fallback implementation)")
    return ctypes.CDLL(LIB_PATH)


lib = _load()

i64 = ctypes.c_int64
i64p = ctypes.POINTER(ctypes.c_int64)
vp = ctypes.c_void_p
f32 = ctypes.c_float
f32p = ctypes.POINTER(ctypes.c_float)
u8p = ctypes.POINTER(ctypes.c_uint8)


class ReplicaOut(ctypes.Structure):
    # output array addresses as plain integers (filled by the C++ kernel)
    _fields_ = [(n, ctypes.c_void_p) for n in (
        "task_stage", "task_kind", "task_mb", "task_start", "task_end",
        "msg_send", "msg_grant", "msg_arrive", "msg_boundary", "msg_dir", "msg_mb",
        "last_bwd_end", "peak_stash", "peak_sets", "peak_mem")] + [
        ("n_tasks", i64), ("n_msgs", i64), ("makespan", i64)]


def _sig(name, argtypes, restype=ctypes.c_int):
    fn = getattr(lib, name)
    fn.argtypes = argtypes
    fn.restype = restype
    return fn


_sig("vp_version", [], ctypes.c_char_p)
# array arguments are passed as raw addresses (ptr() below): building a
# ctypes POINTER object per array cost more than the C++ kernels themselves
_vp = ctypes.c_void_p
_sig("vp_varuna_schedule", [i64, i64, i64, i64, i64, i64, _vp, _vp, _vp])
_sig("vp_gpipe_schedule", [i64, i64, i64, _vp, _vp, _vp])
_sig("vp_run_replica", [i64, i64] + [_vp] * 12 + [ctypes.c_int, ctypes.c_int,
                                                   ctypes.POINTER(ReplicaOut)])
_sig("vp_assign_stages", [i64, _vp, _vp, i64, ctypes.c_double, _vp])
_sig("vp_identify_cutpoints", [i64, _vp, _vp, _vp, i64, ctypes.c_double, _vp])


class VpipeError(RuntimeError):
    pass


def check(rc: int, what: str = "vpipe"):
    """Map a C-ABI status to the reference's exception conventions
    (ConfigError for malformed input, InfeasibleError for no answer,
    RuntimeError for deadlock / CUDA failures)."""
    if rc == VP_OK:
        return
    if rc == VP_ERR_ARGS:
        raise ConfigError(f"{what}: invalid arguments")
    if rc == VP_ERR_INFEASIBLE:
        raise InfeasibleError(f"{what}: infeasible")
    if rc == VP_ERR_DEADLOCK:
        raise RuntimeError(f"{what}: simulation deadlocked")
    if rc == VP_ERR_NOMEM:
        raise MemoryError(what)
    if rc == VP_ERR_UNSUPPORTED:
        raise VpipeError(f"{what}: unsupported shape/layout")
    if rc > 0:
        raise VpipeError(f"{what}: CUDA error {rc}")
    raise VpipeError(f"{what}: error {rc}")


def ptr(arr):
    """Address of a C-contiguous numpy array's data (the array must stay
    alive for the call)."""
    return arr.__array_interface__["data"][0]

"""ctypes binding of libgeek.so (include/geek.h) and device-buffer helpers.

There is no CPU fallback: every compute entry point goes through this
module, and `lib()` raises if the library is missing or no CUDA device is
visible.  Torch tensors are used only as device buffers; the current torch
stream is handed to every call so the kernels are stream-ordered with the
caller's work.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np
import torch

from .errors import EngineError, InvalidInput

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgeek.so")

GEEK_OK, GEEK_EINVAL, GEEK_ECUDA, GEEK_ENOMEM, GEEK_ERANGE = 0, -1, -2, -3, -4
NONE32 = 0xFFFFFFFF

u8p = C.c_void_p
vp = C.c_void_p
u64 = C.c_uint64
i32 = C.c_int


class PermT(C.Structure):
    """geek_perm_t (include/geek.h)."""

    _fields_ = [
        ("u", C.c_uint64),
        ("mask", C.c_uint32), ("c1", C.c_uint32), ("c2", C.c_uint32), ("a1", C.c_uint32),
        ("s1", C.c_uint32), ("s2", C.c_uint32), ("c1inv", C.c_uint32), ("c2inv", C.c_uint32),
        ("table", C.c_uint32), ("inv_table", C.c_uint32),
    ]


# name -> (restype, argtypes)
_SIGS = {
    "geek_version": (i32, []),
    "geek_last_error": (C.c_char_p, []),
    "geek_device_sms": (i32, []),
    "geek_perm_forward": (i32, [vp, i32, vp, vp, u64, vp, vp]),
    "geek_perm_inverse": (i32, [vp, i32, vp, vp, u64, vp, vp]),
    "geek_set_minhash": (i32, [vp, i32, vp, vp, vp, u64, vp, vp]),
    "geek_silk_invscan": (i32, [vp, u64, i32, u64, vp, i32, vp, vp, vp, vp, vp]),
    "geek_project_keys": (i32, [vp, i32, u64, i32, vp, i32, vp, vp, vp]),
    "geek_project_keys_routed": (i32, [vp, i32, u64, i32, vp, i32, vp, i32, u64, u64, vp, vp, i32, vp, vp]),
    "geek_split_plan": (i32, [u64, vp, vp]),
    "geek_coarse_hist": (i32, [vp, u64, i32, i32, vp, vp]),
    "geek_fine_layout": (i32, [vp, i32, u64, vp, vp, vp, vp]),
    "geek_rank_split_counted": (i32, [vp, u64, i32, u64, vp, vp, vp, vp, vp]),
    "geek_rank_split": (i32, [vp, u64, i32, u64, vp, vp, vp]),
    "geek_split_boundary_workspace": (u64, [u64, u64]),
    "geek_split_boundary_stats": (i32, [vp, u64, i32, u64, vp, u64, vp, C.c_double, C.c_double, vp, vp, u64, vp,
                                        u64, vp]),
    "geek_rank_split_strided": (i32, [vp, u64, u64, vp, u64, u64, vp]),
    "geek_column_keys": (i32, [vp, i32, u64, u64, u64, vp, vp]),
    "geek_group_rows": (i32, [vp, u64, i32, vp, vp, vp, vp, vp]),
    "geek_emit_members_codes": (i32, [vp, u64, i32, u64, vp, vp, vp, vp, u64, vp, vp]),
    "geek_majority_vote": (i32, [vp, vp, u64, vp, u64, u64, vp, vp, vp, vp]),
    "geek_emit_winners_codes": (i32, [vp, u64, i32, u64, vp, vp, vp, vp, vp, u64, vp, vp]),
    "geek_group_winners": (i32, [vp, vp, u64, u64, u64, u64, vp, vp, vp, vp]),
    "geek_pick_representatives": (i32, [vp, vp, vp, vp, u64, vp, vp]),
    "geek_sort_groups": (i32, [vp, vp, u64, vp, vp]),
    "geek_exponent_range": (i32, [vp, i32, u64, i32, vp, vp]),
    "geek_exact_sums": (i32, [vp, i32, u64, i32, u64, vp, vp, u64, i32, i32, vp, vp, vp]),
    "geek_sum_pack_bytes": (i32, [vp, u64, i32, i32, i32, vp, vp]),
    "geek_round_means": (i32, [vp, vp, u64, i32, i32, i32, vp, vp]),
    "geek_assign_l2_workspace_size": (u64, [u64, i32, u64]),
    "geek_assign_l2": (i32, [vp, i32, u64, i32, vp, u64, vp, vp, vp, vp, vp, vp, u64, vp]),
    "geek_tc_selftest": (i32, [C.c_uint32, C.c_uint32, i32, vp]),
    "geek_radii_sizes": (i32, [vp, vp, u64, u64, vp, vp, vp]),
    "geek_pairwise_sum": (i32, [vp, u64, vp, vp]),
    "geek_assign_categorical": (i32, [vp, u64, i32, vp, u64, vp, vp, vp]),
    "geek_assign_sparse": (i32, [vp, vp, u64, u64, vp, u64, vp, vp, vp]),
    "geek_doph_reduce": (i32, [vp, vp, vp, vp, u64, u64, u64, vp, vp, vp, vp]),
    "geek_mode_counts": (i32, [vp, u64, i32, u64, u64, vp, vp, u64, vp, vp]),
    "geek_sparse_counts": (i32, [vp, vp, u64, u64, u64, vp, vp, u64, vp, vp]),
    "geek_label_sums": (i32, [vp, i32, u64, i32, vp, vp, u64, i32, i32, vp, vp]),
    "geek_label_mode_counts": (i32, [vp, u64, i32, vp, u64, u64, vp, vp]),
    "geek_label_sparse_counts": (i32, [vp, vp, u64, vp, u64, u64, vp, vp]),
    "geek_unpack_vecs": (i32, [vp, u64, i32, i32, vp, vp, vp]),
    "geek_pack_buckets": (i32, [vp, vp, vp, i32, u64, u64, vp, vp]),
}

_lock = threading.Lock()
_lib = None


def load_library(path: str = LIB_PATH):
    """Load libgeek.so and bind every symbol (no GPU needed)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise EngineError(
                    f"libgeek.so not built at {path}; run `python -m paper_2106_10515_b200._build`")
            L = C.CDLL(path)
            for name, (res, args) in _SIGS.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def lib():
    """The bound library, after checking that a CUDA device is usable."""
    L = load_library()
    if not torch.cuda.is_available():
        raise EngineError("no CUDA device visible: the GEEK B200 kernels have no CPU fallback")
    return L


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise EngineError("no CUDA device visible: the GEEK B200 kernels have no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def check(status: int, what: str = ""):
    if status == GEEK_OK:
        return
    msg = (_lib.geek_last_error() or b"").decode(errors="replace")
    if status == GEEK_EINVAL:
        raise InvalidInput(f"{what}: {msg}" if what else msg)
    raise EngineError(f"{what} failed ({status}): {msg}")


class CallTimer:
    """Brackets every libgeek entry point with CUDA events on the current
    stream (bench.py uses it to time the dominant kernel live)."""

    def __init__(self):
        self.events = []

    def ms_by_name(self):
        torch.cuda.synchronize()
        out = {}
        for name, a, b in self.events:
            s = out.setdefault(name, [0.0, 0])
            s[0] += a.elapsed_time(b)
            s[1] += 1
        return out


_timer = None


def set_call_timer(t):
    global _timer
    _timer = t


def call(name: str, *args):
    L = lib()
    if _timer is not None:
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        st = getattr(L, name)(*args)
        b.record()
        _timer.events.append((name, a, b))
        check(st, name)
        return
    check(getattr(L, name)(*args), name)


def ptr(t) -> C.c_void_p:
    if t is None:
        return C.c_void_p(None)
    if isinstance(t, torch.Tensor):
        if not t.is_cuda:
            raise EngineError("expected a CUDA tensor")
        if not t.is_contiguous():
            raise EngineError("expected a contiguous tensor")
        return C.c_void_p(t.data_ptr())
    raise TypeError(type(t))


def hptr(a: np.ndarray) -> C.c_void_p:
    return a.ctypes.data_as(C.c_void_p)


def empty(n, dtype) -> torch.Tensor:
    return torch.empty(n, dtype=dtype, device=device())


def zeros(n, dtype) -> torch.Tensor:
    return torch.zeros(n, dtype=dtype, device=device())


def to_dev(a, dtype=None) -> torch.Tensor:
    """Host numpy / list -> contiguous device tensor."""
    if isinstance(a, torch.Tensor):
        t = a if a.is_cuda else a.to(device())
        if dtype is not None and t.dtype != dtype:
            t = t.to(dtype)
        return t.contiguous()
    arr = np.ascontiguousarray(a)
    t = torch.from_numpy(arr)
    if dtype is not None:
        t = t.to(dtype)
    # through a (cached) pinned staging copy: the upload is stream-ordered and
    # the host does not wait for the queued kernels, as a pageable copy would
    dev = device()  # (raises EngineError without a GPU before any pinned allocation)
    return t.pin_memory().to(dev, non_blocking=True).contiguous()


def dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return 0
    if t.dtype == torch.float64:
        return 1
    raise InvalidInput(f"unsupported dense dtype {t.dtype}")


# u32 tensors: torch has uint32 with limited op support; we use int32 storage
# and reinterpret (same bits) where the kernels expect uint32.
U32 = torch.int32

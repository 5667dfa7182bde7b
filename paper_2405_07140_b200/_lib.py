"""ctypes binding of include/edgebatch_b200.h (the drop-in C ABI).

The library is loaded from this package directory.  There is no CPU
fallback: if ``libedgebatch_b200.so`` is missing or no CUDA device is present
every entry point raises ``EdgebatchNativeError``.
"""
from __future__ import annotations

import ctypes as C
import os
import sys
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# EB_LIB_PATH: an alternative build of the same library (tools/variants.sh
# launch-bound experiments); the default is the in-tree build
LIB_PATH = os.environ.get("EB_LIB_PATH") or os.path.join(HERE, "libedgebatch_b200.so")

ABI_VERSION = 2        # include/edgebatch_b200.h EB_ABI_VERSION
EB_MAX_K = 64
EB_MAX_CLASSES = 16
EB_N_METRICS = 8
EB_MEM_HOST = 0
EB_MEM_DEVICE = 1

# eb_status
OK = 0
ERR_INVALID_ARG = 1
ERR_CUDA = 2
ERR_K_TOO_LARGE = 3
ERR_TOO_MANY_CLASSES = 4
ERR_NO_DEVICE = 5
ERR_WEIGHTS_DO_NOT_FIT = 10
ERR_UPLINK_EFF_ZERO = 11
ERR_DOWNLINK_EFF_ZERO = 12
ERR_OFF_LADDER = 13
ERR_REVERIFY = 14
ERR_DUPLICATE_ID = 15
ERR_CAP_EXCEEDED = 16
ERR_OVERFLOW = 17
ERR_BAD_MODE = 18
ERR_PADDED_TOO_SMALL = 19
ERR_NONPOSITIVE_LINK = 20
ERR_NAN_INPUT = 21

MET_UP_SUM, MET_DN_SUM, MET_MEM_POOLPAD, MET_LAT_POOLPAD, MET_MEM_BATCHPAD, MET_LAT_BATCHPAD, \
    MET_PADDED, MET_WIN_D = range(8)


class EdgebatchNativeError(RuntimeError):
    """The CUDA library is unavailable or a CUDA call failed."""


class eb_context(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("layers", "hidden_dim", "head_count", "head_dim", "ffn_dim",
                                          "bytes_per_param")] + \
               [(n, C.c_double) for n in ("alpha", "beta", "delta_ppl", "uplink_band_hz", "downlink_band_hz",
                                          "downlink_power_w", "noise_density_w_hz", "uplink_slot_s",
                                          "downlink_slot_s")] + \
               [("bits_per_token", C.c_int64), ("flops_per_s", C.c_double), ("memory_bytes", C.c_double),
                ("gpu_count", C.c_int64), ("has_slot_cap", C.c_int64), ("slot_cap_s", C.c_double)]


CTX_FIELDS = [f[0] for f in eb_context._fields_]
# numpy mirror of eb_context (all 8-byte fields, no padding)
CTX_DTYPE = np.dtype([(n, np.int64 if t is C.c_int64 else np.float64) for n, t in eb_context._fields_])
assert CTX_DTYPE.itemsize == C.sizeof(eb_context) == 8 * len(CTX_FIELDS)


class eb_requests(C.Structure):
    _fields_ = [("id", C.c_void_p), ("prompt_tokens", C.c_void_p), ("output_tokens", C.c_void_p),
                ("deadline_s", C.c_void_p), ("waiting_s", C.c_void_p), ("tolerance", C.c_void_p),
                ("channel_gain", C.c_void_p), ("uplink_power_w", C.c_void_p)]


class eb_batch(C.Structure):
    _fields_ = [("n_inst", C.c_int64), ("n_req", C.c_int64), ("offsets", C.c_void_p), ("ctx_index", C.c_void_p),
                ("req", eb_requests), ("k_max", C.c_int32), ("_pad", C.c_int32)]


class eb_requests_packed(C.Structure):
    _fields_ = [("id", C.c_void_p), ("prompt_tokens", C.c_void_p), ("output_tokens", C.c_void_p),
                ("deadline_s", C.c_void_p), ("waiting_s", C.c_void_p), ("channel_gain", C.c_void_p),
                ("uplink_power_w", C.c_void_p), ("uplink_power_uniform", C.c_int32), ("n_dict", C.c_int32),
                ("token_codes", C.c_void_p), ("prompt_dict", C.c_int32 * 16), ("output_dict", C.c_int32 * 16)]


class eb_batch_packed(C.Structure):
    _fields_ = [("n_inst", C.c_int64), ("n_req", C.c_int64), ("offsets", C.c_void_p), ("ctx_index", C.c_void_p),
                ("req", eb_requests_packed), ("k_max", C.c_int32), ("_pad", C.c_int32)]


class eb_search_params(C.Structure):
    _fields_ = [("pruning", C.c_int32), ("inclusive_bound", C.c_int32), ("exact_tau", C.c_int32),
                ("collect_trajectory", C.c_int32), ("ladder_len", C.c_int32),
                ("ladder", C.c_int32 * EB_MAX_CLASSES), ("algorithm", C.c_int32),
                ("exhaustive_counts", C.c_int32)]


class eb_dftsp_result(C.Structure):
    _fields_ = [("status", C.c_void_p), ("error_index", C.c_void_p), ("z_found", C.c_void_p),
                ("nodes_visited", C.c_void_p), ("nodes_pruned", C.c_void_p), ("n_classes", C.c_void_p),
                ("counts", C.c_void_p), ("class_lengths", C.c_void_p), ("solution", C.c_void_p),
                ("metrics", C.c_void_p), ("traj_offsets", C.c_void_p), ("traj", C.c_void_p),
                ("traj_len", C.c_void_p), ("solution_mask", C.c_void_p)]


P = C.c_void_p
I32, I64, F64 = C.c_int32, C.c_int64, C.c_double
_SIGS = {
    "eb_abi_version": (I32, []),
    "eb_status_string": (C.c_char_p, [I32]),
    "eb_last_error": (C.c_char_p, []),
    "eb_handle_create": (I32, [I32, C.POINTER(P)]),
    "eb_handle_destroy": (I32, [P]),
    "eb_handle_set_stream": (I32, [P, P]),
    "eb_synchronize": (I32, [P]),
    "eb_kernel_launches": (I64, [P]),
    "eb_probe_peaks": (I32, [P, P, P]),
    "eb_dftsp_batch": (I32, [P, P, I32, P, P, P, I32]),
    "eb_dftsp_batch_packed": (I32, [P, P, I32, P, P, P, I32]),
    "eb_dfs_single": (I32, [P, I32, I32, P, P, P, P, P, P, P, P, I64, I32, F64, P, P, P, P, P]),
    "eb_exhaustive_batch": (I32, [P, P, I32, P, I32, P, P, P, P, P, I32]),
    "eb_exhaustive_level_range": (I32, [P, P, I32, P, I32, I64, I64, P]),
    "eb_exhaustive_live_levels": (I32, [P, P, I32, P, P]),
    "eb_exhaustive_counters": (I32, [P, P]),
    "eb_check_direct_batch": (I32, [P, P, I32, P, I64, I64, P, P, P, P, P, P, P, I32]),
    "eb_check_knapsack_batch": (I32, [P, I64, P, P, P, P, P, P, P, P, P, I32]),
    "eb_coefficients_batch": (I32, [P, P, I32, P, P, P, P, P, P, I32]),
    "eb_link_batch": (I32, [P, P, I32, P, I64, P, P, P, I32]),
    "eb_admission_batch": (I32, [P, P, I32, P, I32, I32, P, P, I32]),
    "eb_batch_cost_batch": (I32, [P, P, I32, I64, P, P, P, P, P, P, P, I32]),
    "eb_static_batch_size_batch": (I32, [P, P, I32, P, P, P, P, I32]),
    "eb_stb_batch": (I32, [P, P, I32, P, P, I32, P, P, I32]),
    "eb_nob_batch": (I32, [P, P, I32, P, P, I32, P, I32, P, P, P, P, P, I32]),
}
EXPORTED_SYMBOLS = tuple(_SIGS)

_lib = None
_lib_lock = threading.Lock()
_tls = threading.local()


def load(path: str | None = None):
    """Load the CUDA library (no GPU needed just to load it)."""
    global _lib
    with _lib_lock:
        if _lib is not None and path is None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise EdgebatchNativeError(
                f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        lib = C.CDLL(p)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.eb_abi_version() != ABI_VERSION:
            raise EdgebatchNativeError("ABI version mismatch")
        if path is None:
            _lib = lib
        return lib


def status_string(code: int) -> str:
    return load().eb_status_string(int(code)).decode()


def check(code: int, what: str = "") -> None:
    if code != OK:
        lib = load()
        detail = lib.eb_last_error().decode()
        raise EdgebatchNativeError(f"{what}: {status_string(code)} ({code}) {detail}".strip())


class Handle:
    """Owns an eb_handle (device, stream, scratch)."""

    def __init__(self, device: int = 0):
        self.lib = load()
        h = P()
        code = self.lib.eb_handle_create(int(device), C.byref(h))
        if code != OK:
            raise EdgebatchNativeError(
                f"eb_handle_create(device={device}) failed: {status_string(code)}: "
                f"{self.lib.eb_last_error().decode()}")
        self.ptr = h
        self.device = device

    def launches(self) -> int:
        return int(self.lib.eb_kernel_launches(self.ptr))

    def set_stream(self, stream_ptr: int) -> None:
        check(self.lib.eb_handle_set_stream(self.ptr, P(stream_ptr)), "eb_handle_set_stream")

    def synchronize(self) -> None:
        check(self.lib.eb_synchronize(self.ptr), "eb_synchronize")

    def close(self) -> None:
        if getattr(self, "ptr", None):
            self.lib.eb_handle_destroy(self.ptr)
            self.ptr = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass


def default_device() -> int:
    """The calling process's GPU: torch's current device once torch has
    initialised CUDA, else LOCAL_RANK (one process per GPU under torchrun),
    else 0."""
    torch = sys.modules.get("torch")
    if torch is not None:
        try:
            if torch.cuda.is_initialized():
                return int(torch.cuda.current_device())
        except Exception:
            pass
    return int(os.environ.get("LOCAL_RANK", "0"))


def handle(device: int | None = None) -> Handle:
    """Per-thread default handle (the library keeps no global mutable state)."""
    dev = default_device() if device is None else device
    hs = getattr(_tls, "handles", None)
    if hs is None:
        hs = _tls.handles = {}
    if dev not in hs:
        hs[dev] = Handle(dev)
    return hs[dev]


def ptr(a) -> int | None:
    """Address of a numpy array or torch tensor (None passes NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"], "arrays must be C-contiguous"
        return a.ctypes.data
    return int(a.data_ptr())  # torch.Tensor

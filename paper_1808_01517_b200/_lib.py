"""ctypes binding of libdelimit_sm100a.so (the C ABI in include/delimit.h).

The library is the only compute path: if it is missing or the device is not
sm_100a every op raises DeviceError.  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import DeviceError

LIB_PATH = os.environ.get("DELIMIT_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                          "libdelimit_sm100a.so")

_c_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_int = ctypes.c_int
_size = ctypes.c_size_t

# name -> (restype, argtypes); must match include/delimit.h
SIGNATURES = {
    "dl_abi_version": (_int, []),
    "dl_last_error": (ctypes.c_char_p, []),
    "dl_device_supported": (_int, []),
    "dl_last_launch_count": (_int, []),
    "dl_total_launch_count": (_i64, []),
    "dl_chan_contract_f32": (_int, [_c_p, _c_p, _c_p, _c_p, _i64, _i64, _i64, _i64, _i64, _i64, _i64, _int, _c_p]),
    "dl_lsc_build_operator_f32": (_int, [_c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _i64, _i64, _i64, _i64, _i64, _c_p]),
    "dl_lsc_wgrad_workspace_bytes": (_size, [_i64, _i64, _i64, _i64]),
    "dl_lsc_wgrad_f32": (_int, [_c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _i64, _i64, _i64, _i64, _i64, _i64,
                                _i64, _i64, _i64, _c_p]),
    "dl_chain_supported": (_int, [_i64] * 6 + [_int]),
    "dl_chain_split_terms": (_int, []),
    "dl_chain_mid_bytes": (_size, [_i64] * 4),
    "dl_chain_workspace_bytes": (_size, [_i64] * 8),
    "dl_chain_state_bytes": (_size, []),
    "dl_chain_fwd_f32": (_int, [_c_p, _c_p, _c_p, _c_p, _int, _c_p, _c_p, _c_p, _c_p, _c_p] + [_i64] * 8 + [_c_p]),
    "dl_chain_bwd_f32": (_int, [_c_p] * 7 + [_int] + [_c_p] * 6 + [_i64] * 9 + [_c_p]),
    "dl_debug_chain_prof": (None, [_c_p]),
    "dl_ktimer_arm": (_int, [_int]),
    "dl_ktimer_count": (_i64, [_int]),
    "dl_ktimer_read": (_int, [_int, _int, _c_p]),
    "dl_chain_bwd_gram_f64": (_int, [_c_p] * 6 + [_int] + [_c_p] * 4 + [_i64] * 8 + [_c_p]),
    "dl_chain_gram_dims": (_int, [_i64] * 4 + [_c_p, _c_p]),
    "dl_chain_fwd_mse_f32": (_int, [_c_p] * 5 + [_int] + [_c_p] * 6 + [_i64] * 8 + [_c_p]),
    "dl_chain_mse_supported": (_int, [_i64] * 6 + [_int]),
    "dl_normalize_b0_workspace_bytes": (_size, [_i64] * 3),
    "dl_normalize_b0_f32": (_int, [_c_p, _int] + [_i64] * 7 + [ctypes.c_double] * 2
                            + [_c_p, _i64, _c_p, _i64, _c_p, _c_p, _c_p, _c_p]),
    "dl_chain_fwd_raw_f32": (_int, [_c_p, _int, _i64] + [_c_p] * 5 + [_int] + [_c_p] * 5 + [_i64] * 7 + [_c_p]),
    "dl_round_trip_workspace_bytes": (_size, [_i64] * 6),
    "dl_round_trip_fwd_f32": (_int, [_c_p, _c_p, _c_p, _int, _c_p, _c_p, _c_p] + [_i64] * 6 + [_c_p]),
    "dl_round_trip_bwd_f32": (_int, [_c_p, _c_p, _c_p, _int, _c_p, _c_p, _c_p] + [_i64] * 6 + [_c_p]),
    "dl_gemm_f64": (_int, [_i64, _i64, _i64, _c_p, _i64, _int, _c_p, _i64, _int, _c_p, _i64, ctypes.c_double,
                            ctypes.c_double, _c_p]),
    "dl_lsc_dw_from_dl_f64": (_int, [_c_p, _c_p, _c_p] + [_i64] * 5 + [_c_p]),
    "dl_b0_voxel_scale_f32": (_int, [_c_p, _int] + [_i64] * 7 + [ctypes.c_double] * 2
                              + [_c_p, _i64, _c_p, _c_p, _c_p, _c_p, _c_p]),
}

_lock = threading.Lock()
_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load (once) and type the library.  Raises DeviceError if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise DeviceError(f"{os.path.basename(path)} is not built (run __graft_entry__.build()); "
                                  "the sm_100a CUDA path is the only implementation")
            lib = ctypes.CDLL(path)
            for name, (res, args) in SIGNATURES.items():
                # an A/B build of an older source (DELIMIT_LIB) may lack newer entry points; the product library
                # exports every one (tests/test_abi.py)
                fn = getattr(lib, name, None) if os.environ.get("DELIMIT_LIB") else getattr(lib, name)
                if fn is None:
                    continue
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def last_error() -> str:
    msg = load().dl_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str) -> None:
    if status != 0:
        raise DeviceError(f"{what}: {last_error()} (status {status})")


def call(name: str, *args) -> None:
    """Call a status-returning entry point and raise DeviceError on failure."""
    check(getattr(load(), name)(*args), name)


def launch_count() -> int:
    return int(load().dl_last_launch_count())


def ktimer_arm(on: bool = True) -> None:
    """Bracket the fused chain kernel's fp16-pass launches with CUDA events (see dl_ktimer_arm)."""
    call("dl_ktimer_arm", int(on))


def ktimer_count(slot: int) -> int:
    """Launches bracketed so far in a slot (0 forward chain, 1 adjoint chain, 2 Gram)."""
    return int(load().dl_ktimer_count(slot))


def ktimer_read(slot: int, back: int = 0) -> float:
    """Duration (ms) of a bracketed launch: slot 0 forward chain, 1 adjoint chain, 2 Gram; back = 0 is the last."""
    ms = ctypes.c_float()
    call("dl_ktimer_read", slot, back, ctypes.byref(ms))
    return float(ms.value)


def total_launches() -> int:
    """Kernel launches this library has enqueued since load (for bench.py's gpu_launches)."""
    return int(load().dl_total_launch_count())

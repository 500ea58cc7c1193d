"""ctypes binding of libtfft.so (include/tfft.h).

The product has exactly one compute path: this library. There is no CPU
fallback — if the library or a GPU is missing, every compute call raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TFFT_LIB_PATH") or os.path.join(_HERE, "libtfft.so")  # override: experiments only

TFFT_OK, TFFT_EINVAL, TFFT_ECUDA, TFFT_ENOMEM, TFFT_EUNSUPPORTED, TFFT_EIO = 0, 1, 3, 4, 5, 6
FP32, FP64 = 0, 1
AT_NONE, AT_INPUT, AT_STAGE, AT_OUTPUT = 0, 1, 2, 3
SCHEME_CODE = {"none": 0, "one_sided": 1, "two_sided_thread": 2, "two_sided_group": 3}


class Fault(ctypes.Structure):
    _fields_ = [("signal", ctypes.c_int64), ("element", ctypes.c_int64),
                ("where", ctypes.c_int32), ("stage", ctypes.c_int32),
                ("component", ctypes.c_int32), ("bit", ctypes.c_int32)]


class Flag(ctypes.Structure):
    _fields_ = [("group", ctypes.c_int64), ("signal", ctypes.c_int64),
                ("discrepancy", ctypes.c_double)]


class Report(ctypes.Structure):
    _fields_ = [("groups", ctypes.c_int64), ("recompute_count", ctypes.c_int64),
                ("pass_count", ctypes.c_int64), ("max_rel_discrepancy", ctypes.c_double),
                ("n_flagged", ctypes.c_int64), ("n_corrected", ctypes.c_int64),
                ("n_unrecoverable", ctypes.c_int64),
                ("flagged", ctypes.POINTER(Flag)), ("flagged_cap", ctypes.c_int64),
                ("corrected_group", ctypes.POINTER(ctypes.c_int64)),
                ("corrected_signal", ctypes.POINTER(ctypes.c_int64)),
                ("corrected_cap", ctypes.c_int64),
                ("unrecoverable", ctypes.POINTER(ctypes.c_int64)),
                ("unrecoverable_cap", ctypes.c_int64),
                ("fault_fired", ctypes.c_int32)]


# symbol -> (restype, argtypes); every symbol include/tfft.h declares
_VP, _I64, _INT, _DBL = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
SIGNATURES = {
    "tfft_plan_create": (_INT, [ctypes.POINTER(_VP), _I64, _INT, _INT, ctypes.POINTER(_I64), _I64, _INT]),
    "tfft_plan_destroy": (_INT, [_VP]),
    "tfft_execute": (_INT, [_VP, _VP, _VP, _I64, _INT, _VP]),
    "tfft_run_protected": (_INT, [_VP, _VP, _VP, _I64, _INT, _DBL, _DBL, _VP, _VP,
                                  ctypes.POINTER(Fault), _INT, ctypes.POINTER(Report), _VP]),
    "tfft_run_protected_host": (_INT, [_VP, _VP, _VP, _I64, _INT, _DBL, _DBL, _VP, _VP,
                                       ctypes.POINTER(Fault), _INT, ctypes.POINTER(Report), _VP]),
    "tfft_signal_file_batch": (_INT, [ctypes.c_char_p, _I64, _INT, ctypes.POINTER(_I64)]),
    "tfft_run_protected_file": (_INT, [_VP, ctypes.c_char_p, ctypes.c_char_p, _INT, _DBL, _DBL, _VP, _VP,
                                       ctypes.POINTER(Fault), _INT, ctypes.POINTER(_I64),
                                       ctypes.POINTER(Report), _VP]),
    "tfft_run_campaign": (_INT, [_VP, _VP, _VP, _I64, _I64, _INT, _DBL, _DBL, _VP, _VP,
                                 ctypes.POINTER(Fault), _INT, ctypes.POINTER(ctypes.c_double),
                                 ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(Report), _VP]),
    "tfft_protect_launch": (_INT, [_VP, _VP, _VP, _I64, _INT, _DBL, _DBL, _VP, _VP,
                                   ctypes.POINTER(Fault), _INT, ctypes.POINTER(Report), _VP]),
    "tfft_protect_finish": (_INT, [_VP, _VP, _VP, _I64, _INT, _DBL, _DBL, _VP, _VP, _INT,
                                   ctypes.POINTER(Report), _VP]),
    "tfft_set_check_level": (_INT, [_VP, _INT]),
    "tfft_set_device_correction": (_INT, [_VP, _INT]),
    "tfft_plan_exec_passes": (_INT, [_VP]),
    "tfft_tile_fft": (_INT, [_VP, _VP, _I64, _I64, _INT, _INT, _INT, _VP]),
    "tfft_encode_group": (_INT, [_VP, _VP, _I64, _VP, _VP, _VP, _VP, _VP, _VP]),
    "tfft_detect": (_INT, [_VP, _VP, _I64, _VP, _VP, _VP, _DBL, _DBL, _VP, _VP, _VP]),
    "tfft_correct_signal": (_INT, [_VP, _VP, _VP, _I64, _I64, _VP, _INT, _VP]),
    "tfft_element_encode": (_INT, [_INT, _I64, _VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "tfft_element_verify": (_INT, [_INT, _I64, _VP, _VP, _VP, _VP, _VP, _DBL, _DBL, _VP,
                                   ctypes.POINTER(ctypes.c_int32), _VP]),
    "tfft_flip_bit": (_INT, [_VP, _I64, _INT, _INT, _VP]),
    "tfft_execute_stage": (_INT, [_VP, _INT, _VP, _VP, _I64, _INT, _VP]),
    "tfft_scale": (_INT, [_VP, _I64, _INT, _DBL, _VP]),
    "tfft_tune_variants": (_INT, [_INT, _INT]),
    "tfft_tune_select": (_INT, [_INT, _INT, _INT]),
    "tfft_tune_pass_variants": (_INT, [_INT, _INT]),
    "tfft_tune_pass_select": (_INT, [_INT, _INT, _INT, _INT]),
    "tfft_report_fetch": (_INT, [_VP, ctypes.POINTER(Report)]),
    "tfft_dft": (_INT, [_VP, _VP, _I64, _I64, _INT, _VP]),
    "tfft_launch_count": (_INT, [ctypes.POINTER(_I64)]),
    "tfft_last_error": (ctypes.c_char_p, []),
    "tfft_version": (_INT, []),
}

_lib = None
_lock = threading.Lock()


def load():
    """Load libtfft.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_2405_02520_b200.build` "
                    "(there is no CPU fallback)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


class TfftError(RuntimeError):
    pass


def check(rc: int, what: str = ""):
    if rc == TFFT_OK:
        return
    msg = load().tfft_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == TFFT_EINVAL:
        raise ValueError(text)
    if rc == TFFT_ENOMEM:
        raise MemoryError(text)
    if rc == TFFT_EUNSUPPORTED:
        raise NotImplementedError(text)
    if rc == TFFT_EIO:
        raise OSError(text)
    raise TfftError(text)


def launch_count() -> int:
    """Kernels libtfft.so has launched in this process (tfft_launch_count)."""
    c = ctypes.c_int64()
    check(load().tfft_launch_count(ctypes.byref(c)), "tfft_launch_count")
    return int(c.value)

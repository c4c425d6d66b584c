"""ctypes binding of libomega_b200.so (include/ob_api.h).

The product path has no CPU fallback: importing this module without the
built library raises ImportError with the build command.  Status codes map
to the reference's exception types.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# OB_LIB_VARIANT=name loads libomega_b200.<name>.so from the package directory instead
# (same-box A/B of two builds, tools/ab_variants.sh); the default is the in-tree build
_VARIANT = os.environ.get("OB_LIB_VARIANT", "")
LIB_PATH = os.path.join(_HERE, f"libomega_b200.{_VARIANT}.so" if _VARIANT else "libomega_b200.so")

OB_OK, OB_EINVAL, OB_ENOTFOUND, OB_ECOMM, OB_ECUDA, OB_ENOMEM, OB_ESTATE = range(7)
STRATEGY = {"full": 0, "sampled": 1, "srpe": 2, "srpe-cgp": 3}
MAX_FANOUT = 200  # OB_MAX_FANOUT
MAX_LAYERS = 8
POLICY = {"ratio": 0, "is": 1, "random": 2}
KIND_TAGS = {"gcn": 0, "sage_mean": 1, "gat": 2, "power_mean": 3, "moments": 4, "sage_max": 5}


class TransportError(RuntimeError):
    """Collective failure (collectives.py:31)."""


class ObConfig(C.Structure):
    _fields_ = [
        ("device", C.c_int32),
        ("strategy", C.c_int32),
        ("gamma", C.c_double),
        ("policy", C.c_int32),
        ("num_partitions", C.c_int32),
        ("rank", C.c_int32),
        ("seed", C.c_uint64),
        ("stream", C.c_uint64),
        ("nccl_id", C.c_void_p),
        ("num_fanouts", C.c_int32),
        ("fanouts", C.c_int32 * 8),
    ]


class ObLayer(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("in_dim", C.c_int32),
        ("out_dim", C.c_int32),
        ("p", C.c_float),
        ("n", C.c_int32),
    ]


class ObBreakdown(C.Structure):
    _fields_ = [
        ("fetch_ms", C.c_double),
        ("transfer_ms", C.c_double),
        ("compute_ms", C.c_double),
        ("collective_bytes", C.c_int64),
        ("fetch_bytes", C.c_int64),
        ("num_candidates", C.c_int64),
        ("num_targets", C.c_int64),
        ("h2d_bytes", C.c_int64),
        ("d2h_bytes", C.c_int64),
        ("total_device_ms", C.c_double),
        ("allgather_bytes", C.c_int64),
    ]


_P = C.c_void_p
_I64P = C.POINTER(C.c_int64)
_SIGS = {
    "ob_last_error": (C.c_char_p, []),
    "ob_version": (C.c_int, []),
    "ob_engine_create": (C.c_int, [C.POINTER(ObConfig), C.POINTER(_P)]),
    "ob_engine_destroy": (C.c_int, [_P]),
    "ob_load_graph": (C.c_int, [_P, C.c_int64, _P, _P, C.c_int64, _P, C.c_int32]),
    "ob_load_pe": (C.c_int, [_P, C.c_int32, _P, C.c_int64, C.c_int32]),
    "ob_generate_graph": (C.c_int, [_P, C.c_int64, C.c_double, C.c_double, C.c_int32, C.c_uint64]),
    "ob_generate_pe": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_uint64]),
    "ob_graph_info": (C.c_int, [_P, _I64P, _I64P, _I64P, _I64P]),
    "ob_graph_csr": (C.c_int, [_P, C.c_int32, _P, _P, _P]),
    "ob_read_rows": (C.c_int, [_P, C.c_int32, C.c_int64, _P, _P]),
    "ob_load_model": (C.c_int, [_P, C.c_int32, C.POINTER(ObLayer), C.POINTER(C.c_void_p)]),
    "ob_precompute_pe": (C.c_int, [_P]),
    "ob_read_pe": (C.c_int, [_P, C.c_int32, _P]),
    "ob_serve": (C.c_int, [_P, C.c_int32, _P, C.c_int64, _P, _P, C.POINTER(ObBreakdown)]),
    "ob_serve_device": (C.c_int, [_P, C.c_int32, _P, C.c_int64, _P, _P, C.POINTER(ObBreakdown)]),
    "ob_serve_submit": (C.c_int, [_P, C.c_int32, _P, C.c_int64, _P, _P, C.POINTER(C.c_int64)]),
    "ob_serve_i32": (C.c_int, [_P, C.c_int32, _P, C.c_int64, _P, _P, C.POINTER(ObBreakdown)]),
    "ob_serve_submit_i32": (C.c_int, [_P, C.c_int32, _P, C.c_int64, _P, _P, C.POINTER(C.c_int64)]),
    "ob_serve_wait": (C.c_int, [_P, C.c_int64, C.POINTER(ObBreakdown)]),
    "ob_set_lanes": (C.c_int, [_P, C.c_int32]),
    "ob_lanes_fork": (C.c_int, [_P]),
    "ob_lanes_join": (C.c_int, [_P]),
    "ob_last_plan": (C.c_int, [_P, _I64P, _I64P, _P, _P, _P, _P, _P]),
    "ob_last_block_sizes": (C.c_int, [_P, C.c_int32, C.c_int32, _I64P, _I64P, _I64P]),
    "ob_last_block": (C.c_int, [_P, C.c_int32, C.c_int32, _P, _P, _P, _P, _P, _P, _P, _P]),
    "ob_reserve": (C.c_int, [_P, C.c_int32, C.c_int64]),
    "ob_profile": (C.c_int, [_P, C.c_int32]),
    "ob_set_graphs": (C.c_int, [_P, C.c_int32]),
    "ob_profile_read": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_double), _I64P, C.POINTER(C.c_double),
                                  C.POINTER(C.c_double)]),
    "ob_partition_owner": (C.c_int, [_P, _P]),
    "ob_launch_count": (C.c_int64, [_P]),
    "ob_nccl_unique_id": (C.c_int, [_P]),
}
EXPORTED = tuple(_SIGS)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2501_08547_b200.build` "
            "(the serving path has no CPU fallback)"
        )
    # One libnccl per process: pre-load the copy torch is built against (the
    # wheel's nvidia/nccl) so our NEEDED libnccl.so.2 resolves to it whether or
    # not torch is imported before or after us.
    try:
        import nvidia.nccl as _nccl

        for d in _nccl.__path__:
            p = os.path.join(d, "lib", "libnccl.so.2")
            if os.path.exists(p):
                C.CDLL(p, mode=C.RTLD_GLOBAL)
                break
    except ImportError:
        pass
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(status: int) -> None:
    if status == OB_OK:
        return
    msg = lib.ob_last_error().decode(errors="replace")
    if status == OB_EINVAL:
        raise ValueError(msg)
    if status == OB_ENOTFOUND:
        raise KeyError(msg)
    if status == OB_ECOMM:
        raise TransportError(msg)
    raise RuntimeError(f"libomega_b200: {msg} (status {status})")


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)

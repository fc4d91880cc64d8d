"""ctypes binding of libb2m.so (include/b2m.h).

The product path runs ONLY through this native library: there is no CPU or
PyTorch fallback.  If the extension is missing, importing it raises
``NativeLibraryMissing`` with the build command; on a machine without a GPU the
library still loads (its symbols can be inspected) but every compute call
fails with a CUDA error.
"""
from __future__ import annotations

import ctypes as C
import os

from .errors import raise_for_status

HERE = os.path.dirname(os.path.abspath(__file__))
# B2M_LIB lets tools/ experiments load an alternative in-tree build variant
LIB_PATH = os.environ.get("B2M_LIB") or os.path.join(HERE, "libb2m.so")

_dp = C.POINTER(C.c_double)
_u64 = C.c_uint64
_i64 = C.c_int64
_st = C.c_int


class NativeLibraryMissing(ImportError):
    pass


class b2m_grid(C.Structure):
    """Layout-identical to pic::Grid (grid.hpp:15-41), 64 bytes."""
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("pad_", C.c_int32),
                ("lx", C.c_double), ("ly", C.c_double), ("lz", C.c_double),
                ("dx", C.c_double), ("dy", C.c_double), ("dz", C.c_double)]


class b2m_mover_params(C.Structure):
    """Layout-identical to pic::MoverParams (kernels.hpp:30-39), 32 bytes."""
    _fields_ = [("dt", C.c_double), ("qom", C.c_double), ("pc_iterations", C.c_int32),
                ("pad_", C.c_int32), ("beta", C.c_double)]


assert C.sizeof(b2m_grid) == 64 and C.sizeof(b2m_mover_params) == 32

# name -> (restype, argtypes); every symbol include/b2m.h declares
SIGNATURES = {
    "b2m_abi_version": (C.c_int, []),
    "b2m_status_name": (C.c_char_p, [_st]),
    "b2m_last_error": (C.c_char_p, []),
    "b2m_device_count": (C.c_int, []),
    "b2m_launch_count": (_u64, []),
    "b2m_grid_make": (_st, [C.c_int] * 3 + [C.c_double] * 3 + [C.POINTER(b2m_grid)]),
    "b2m_mover_params_make": (_st, [C.c_double, C.c_double, C.c_int,
                                    C.POINTER(b2m_mover_params)]),
    "b2m_move_batch_host": (_st, [C.POINTER(b2m_grid), C.POINTER(b2m_mover_params), _dp, _dp]
                            + [_dp] * 6 + [_u64, C.c_int, C.POINTER(_i64)]),
    "b2m_set_device": (_st, [C.c_int]),
    "b2m_ctx_create": (_st, [C.c_int, C.POINTER(b2m_grid), C.c_int, C.POINTER(_u64), C.c_int,
                             C.POINTER(C.c_void_p)]),
    "b2m_ctx_destroy": (_st, [C.c_void_p]),
    "b2m_ctx_set_stream": (_st, [C.c_void_p, C.c_void_p]),
    "b2m_ctx_set_mode": (_st, [C.c_void_p, C.c_int]),
    "b2m_host_register": (_st, [C.c_void_p, C.c_size_t]),
    "b2m_host_unregister": (_st, [C.c_void_p]),
    "b2m_host_alloc": (_st, [C.c_size_t, C.POINTER(C.c_void_p)]),
    "b2m_host_free": (_st, [C.c_void_p]),
    "b2m_field_upload": (_st, [C.c_void_p, _dp, _dp, _u64]),
    "b2m_field_upload_device": (_st, [C.c_void_p, C.c_void_p, C.c_void_p, _u64]),
    "b2m_field_device_ptrs": (_st, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "b2m_kernel_timing_begin": (_st, [C.c_void_p, C.c_int]),
    "b2m_kernel_timing_read": (_st, [C.c_void_p, C.POINTER(C.c_float), C.c_int,
                                     C.POINTER(C.c_int)]),
    "b2m_species_upload": (_st, [C.c_void_p, C.c_int, C.POINTER(_dp), _u64]),
    "b2m_species_download": (_st, [C.c_void_p, C.c_int, C.POINTER(_dp), _u64, C.POINTER(_u64)]),
    "b2m_species_upload_range": (_st, [C.c_void_p, C.c_int, C.POINTER(_dp), _u64, _u64]),
    "b2m_species_download_range": (_st, [C.c_void_p, C.c_int, C.POINTER(_dp), _u64, _u64]),
    "b2m_species_set_count": (_st, [C.c_void_p, C.c_int, _u64]),
    "b2m_species_count": (_st, [C.c_void_p, C.c_int, C.POINTER(_u64)]),
    "b2m_species_capacity": (_st, [C.c_void_p, C.c_int, C.POINTER(_u64)]),
    "b2m_species_device_ptrs": (_st, [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]),
    "b2m_move": (_st, [C.c_void_p, C.c_int, C.POINTER(b2m_mover_params)]),
    "b2m_move_all": (_st, [C.c_void_p, C.POINTER(b2m_mover_params)]),
    "b2m_move_range": (_st, [C.c_void_p, C.c_int, C.POINTER(b2m_mover_params), _u64, _u64]),
    "b2m_run_mover_host": (_st, [C.c_void_p, C.c_int, C.POINTER(_dp), C.POINTER(_u64),
                                 C.POINTER(b2m_mover_params), _u64]),
    "b2m_sort_species": (_st, [C.c_void_p, C.c_int]),
    "b2m_sync": (_st, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(_i64)]),
    "b2m_field_phase_stub": (_st, [C.c_void_p, C.c_int]),
    "b2m_field_download": (_st, [C.c_void_p, _dp, _dp]),
    "b2m_field_phase_stub_host": (_st, [C.POINTER(b2m_grid), _dp, _dp, C.c_int]),
    "b2m_moments_zero": (_st, [C.c_void_p, C.c_int]),
    "b2m_deposit": (_st, [C.c_void_p, C.c_int, C.c_double]),
    "b2m_move_deposit_all": (_st, [C.c_void_p, C.POINTER(b2m_mover_params),
                                   C.POINTER(C.c_double)]),
    "b2m_moments_download": (_st, [C.c_void_p, C.POINTER(_dp), C.c_int]),
    "b2m_moments_device_ptr": (_st, [C.c_void_p, C.POINTER(_dp), C.POINTER(_u64)]),
    "b2m_deposit_moments_host": (_st, [C.POINTER(b2m_grid)] + [_dp] * 6 +
                                 [_u64, C.c_double, C.c_int, C.POINTER(_dp)]),
    "b2m_event_record": (_st, [C.c_void_p, C.c_int]),
    "b2m_event_elapsed_ms": (_st, [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_float)]),
    "b2m_slab_config": (_st, [C.c_void_p, C.c_int, C.c_int]),
    "b2m_owner_of": (C.c_int, [C.POINTER(b2m_grid), C.c_int, C.c_double]),
    "b2m_move_migrate": (_st, [C.c_void_p, C.c_int, C.POINTER(b2m_mover_params)]),
    "b2m_move_migrate_all": (_st, [C.c_void_p, C.POINTER(b2m_mover_params)]),
    "b2m_outbox": (_st, [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p), C.POINTER(_u64)]),
    "b2m_inbox_append": (_st, [C.c_void_p, C.c_int, C.c_void_p, _u64]),
    "b2m_world_id": (_st, [C.c_void_p]),
    "b2m_world_nccl_available": (_st, []),
    "b2m_world_init": (_st, [C.c_void_p, C.c_void_p, C.c_int, C.c_int]),
    "b2m_world_set_total": (_st, [C.c_void_p, C.POINTER(_u64)]),
    "b2m_world_broadcast_field": (_st, [C.c_void_p, C.c_int]),
    "b2m_world_reduce_moments": (_st, [C.c_void_p]),
    "b2m_world_step": (_st, [C.c_void_p, C.POINTER(b2m_mover_params), C.POINTER(_u64),
                             C.POINTER(_u64)]),
    "b2m_world_loopback_step": (_st, [C.POINTER(C.c_void_p), C.c_int,
                                      C.POINTER(b2m_mover_params), C.POINTER(_u64)]),
    "b2m_gem_counts": (_st, [C.POINTER(b2m_grid), C.c_int, C.POINTER(_u64)]),
    "b2m_gem_species_params": (_st, [C.POINTER(b2m_grid), C.c_int, _dp, _dp]),
    "b2m_gem_fill_species": (_st, [C.POINTER(b2m_grid), C.c_int, _u64, C.c_int, C.POINTER(_dp),
                                   C.c_int]),
    "b2m_gem_fill_species_range": (_st, [C.POINTER(b2m_grid), C.c_int, _u64, C.c_int, _u64, _u64,
                                         C.POINTER(_dp), C.c_int]),
    "b2m_gem_field": (_st, [C.POINTER(b2m_grid), _dp, _dp]),
    "b2m_gem_like_field": (_st, [C.POINTER(b2m_grid), _dp, _dp]),
}

_lib = None


def lib() -> C.CDLL:
    """Load libb2m.so once; raise loudly when it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryMissing(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (or make -C paper_1904_03684_b200/csrc)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.b2m_abi_version() != 1:
            raise NativeLibraryMissing("libb2m.so ABI version mismatch")
        _lib = L
    return _lib


def last_error() -> str:
    return (lib().b2m_last_error() or b"").decode(errors="replace")


def check(status: int) -> None:
    """Raise the reference-taxonomy exception for a non-OK status."""
    if status != 0:
        raise_for_status(status, last_error())


def dptr(a):
    """float64 numpy array -> double*"""
    return a.ctypes.data_as(_dp)


def ptr6(arrs):
    return (_dp * 6)(*[dptr(a) for a in arrs])

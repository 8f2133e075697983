"""ctypes binding of libholosplat.so (include/holosplat.h).

There is no CPU fallback: if the native library or a B200 is missing, every
entry point raises.  The library is built in-tree by
``python -c 'import __graft_entry__ as g; g.build()'`` (or ``make -C
paper_2511_15022_b200/csrc``).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# HOLOSPLAT_LIB: load another build of the same library (A/B timing of two
# builds in one process tree, tools/ab_build.sh); the default is the in-tree build.
LIB_PATH = os.environ.get("HOLOSPLAT_LIB") or os.path.join(_HERE, "libholosplat.so")
CXX_LIB_PATH = os.path.join(_HERE, "libholo_b200.so")

HS_OK, HS_EINVAL, HS_ENONFINITE, HS_ECUDA, HS_ENOMEM, HS_EOVERFLOW = range(6)

_lib = None


class HoloError(RuntimeError):
    """Base error; mirrors the reference's exception split."""


class HoloInvalidArgument(HoloError, ValueError):
    """std::invalid_argument in the reference."""


class HoloNonFinite(HoloError):
    """std::runtime_error("Adan: non-finite gradient in group <g>")."""


class HoloCudaError(HoloError):
    pass


class HoloOverflow(HoloError):
    pass


class hs_prop_spec(C.Structure):
    _fields_ = [("wavelengths", C.POINTER(C.c_double)), ("n_wavelengths", C.c_int),
                ("pixel_pitch", C.c_double), ("pad_factor", C.c_int),
                ("aperture_radius", C.c_double)]


class hs_adan_config(C.Structure):
    _fields_ = [("beta1", C.c_double), ("beta2", C.c_double), ("beta3", C.c_double),
                ("eps", C.c_double)]


class hs_trainer_config(C.Structure):
    _fields_ = [("n", C.c_int), ("c", C.c_int), ("width", C.c_int), ("height", C.c_int),
                ("planes", C.c_int), ("distances", C.POINTER(C.c_double)),
                ("spec", hs_prop_spec), ("total_steps", C.c_int),
                ("h_target", C.POINTER(C.c_float)), ("h_masks", C.POINTER(C.c_uint8)),
                ("plane_begin", C.c_int), ("plane_end", C.c_int), ("channels_total", C.c_int)]


class hs_poh_config(C.Structure):
    _fields_ = [("c", C.c_int), ("height", C.c_int), ("width", C.c_int), ("planes", C.c_int),
                ("distances", C.POINTER(C.c_double)), ("spec", hs_prop_spec),
                ("h_target", C.POINTER(C.c_float)), ("h_masks", C.POINTER(C.c_uint8)), ("steps", C.c_int),
                ("lambda_comp", C.c_double), ("lambda_field", C.c_double), ("lr", C.c_double)]


_SIGS = {
    "hs_trainer_step_host": [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_double)],
    "hs_trainer_run_host": [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_double)],
    "hs_compute_metrics": [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                           C.POINTER(C.c_double), C.POINTER(C.c_double)],
    "hs_dpac_encode": [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p],
    "hs_poh_field": [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p],
    "hs_convert_random_poh_field": [C.c_void_p, C.POINTER(hs_poh_config), C.c_void_p, C.c_void_p,
                                    C.POINTER(C.c_double)],
    "hs_ctx_create": [C.c_int, C.POINTER(C.c_void_p)],
    "hs_ctx_destroy": [C.c_void_p],
    "hs_ctx_set_stream": [C.c_void_p, C.c_void_p],
    "hs_ctx_synchronize": [C.c_void_p],
    "hs_device_alloc": [C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)],
    "hs_device_free": [C.c_void_p, C.c_void_p],
    "hs_copy_h2d": [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t],
    "hs_copy_d2h": [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t],
    "hs_build_tile_index": [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                            C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_int64),
                            C.POINTER(C.c_int)],
    "hs_rasterize_forward": [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p],
    "hs_rasterize_backward": [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                              C.c_void_p],
    "hs_propagate": [C.c_void_p, C.POINTER(hs_prop_spec), C.c_int, C.c_double, C.c_double, C.c_void_p,
                     C.c_int, C.c_int, C.c_int, C.c_void_p],
    "hs_propagate_multi": [C.c_void_p, C.POINTER(hs_prop_spec), C.POINTER(C.c_double), C.c_int,
                           C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p],
    "hs_propagate_multi_backward": [C.c_void_p, C.POINTER(hs_prop_spec), C.POINTER(C.c_double), C.c_int,
                                    C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p],
    "hs_intensity": [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p],
    "hs_loss": [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                C.c_void_p, C.c_void_p, C.POINTER(C.c_double)],
    "hs_build_masks": [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p],
    "hs_adan_step": [C.c_void_p, C.POINTER(hs_adan_config), C.c_char_p, C.c_void_p, C.c_void_p,
                     C.c_void_p, C.c_int64, C.c_int, C.c_double],
    "hs_cosine_lr": [C.c_int, C.c_int, C.c_double, C.c_double, C.POINTER(C.c_double)],
    "hs_trainer_create": [C.c_void_p, C.POINTER(hs_trainer_config), C.POINTER(C.c_void_p)],
    "hs_trainer_destroy": [C.c_void_p],
    "hs_trainer_set_params": [C.c_void_p, C.c_void_p, C.c_int],
    "hs_trainer_get_params": [C.c_void_p, C.c_void_p, C.c_int],
    "hs_trainer_params_ptr": [C.c_void_p],
    "hs_trainer_grads_ptr": [C.c_void_p],
    "hs_trainer_flags_ptr": [C.c_void_p],
    "hs_trainer_param_count": [C.c_void_p],
    "hs_trainer_step": [C.c_void_p, C.POINTER(C.c_double)],
    "hs_trainer_forward_backward": [C.c_void_p],
    "hs_trainer_apply_update": [C.c_void_p],
    "hs_trainer_check_grads": [C.c_void_p],
    "hs_trainer_last_loss": [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int64)],
    "hs_trainer_loss_partials": [C.c_void_p, C.POINTER(C.c_double)],
    "hs_trainer_reserve_pairs": [C.c_void_p, C.c_int64],
    "hs_trainer_use_graph": [C.c_void_p, C.c_int],
    "hs_trainer_set_deterministic": [C.c_void_p, C.c_int],
    "hs_trainer_check_grads_range": [C.c_void_p, C.c_int64, C.c_int64],
    "hs_trainer_apply_update_range": [C.c_void_p, C.c_int64, C.c_int64],
    "hs_ctx_set_deterministic": [C.c_void_p, C.c_int],
    "hs_trainer_set_profiling": [C.c_void_p, C.c_int],
    "hs_trainer_stage_ms": [C.c_void_p, C.POINTER(C.c_double)],
    "hs_trainer_step_count": [C.c_void_p],
    "hs_trainer_set_row_slab": [C.c_void_p, C.c_int, C.c_int],
    "hs_trainer_slab_counts": [C.c_void_p, C.c_int, C.POINTER(C.c_int64)],
    "hs_trainer_slab_send_ptr": [C.c_void_p],
    "hs_trainer_slab_recv_ptr": [C.c_void_p],
    "hs_trainer_slab_stage": [C.c_void_p, C.c_int],
    "hs_trainer_slab_recv2_ptr": [C.c_void_p],
    "hs_trainer_slab_flags_ptr": [C.c_void_p],
    "hs_trainer_slab_set_peers": [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)],
    "hs_trainer_slab_status": [C.c_void_p, C.POINTER(C.c_uint32)],
    "hs_trainer_slab_error_ptr": [C.c_void_p],
    "hs_trainer_slab_forward_backward": [C.c_void_p],
    "hs_comm_unique_id": [C.c_void_p],
    "hs_ctx_comm_init": [C.c_void_p, C.c_void_p, C.c_int, C.c_int],
    "hs_ctx_comm_adopt": [C.c_void_p, C.c_void_p],
    "hs_ctx_comm_info": [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int)],
    "hs_ctx_comm_destroy": [C.c_void_p],
    "hs_trainer_sharded_step": [C.c_void_p, C.POINTER(C.c_double)],
    "hs_ctx_set_tight_binning": [C.c_void_p, C.c_int],
    "hs_random_uniform": [C.c_uint64, C.c_int64, C.c_double, C.c_double, C.c_void_p],
    "hs_ipc_get_handle": [C.c_void_p, C.c_void_p],
    "hs_ipc_open_handle": [C.c_void_p, C.POINTER(C.c_void_p)],
    "hs_ipc_close": [C.c_void_p],
    "hs_last_error": [],
    "hs_kernel_launch_count": [],
}

_RESTYPES = {
    "hs_last_error": C.c_char_p,
    "hs_kernel_launch_count": C.c_uint64,
    "hs_trainer_params_ptr": C.c_void_p,
    "hs_trainer_grads_ptr": C.c_void_p,
    "hs_trainer_flags_ptr": C.c_void_p,
    "hs_trainer_slab_error_ptr": C.c_void_p,
    "hs_trainer_slab_send_ptr": C.c_void_p,
    "hs_trainer_slab_recv_ptr": C.c_void_p,
    "hs_trainer_slab_recv2_ptr": C.c_void_p,
    "hs_trainer_slab_flags_ptr": C.c_void_p,
    "hs_trainer_param_count": C.c_int64,
    "hs_trainer_step_count": C.c_int,
    "hs_ctx_destroy": None,
    "hs_trainer_destroy": None,
}

EXPORTED = tuple(_SIGS)


def load(path: str = LIB_PATH):
    """Loads (once) and returns the native library; raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise HoloError(
            f"native library missing: {path}; build it with __graft_entry__.build() "
            "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, args in _SIGS.items():
        if os.environ.get("HOLOSPLAT_LIB") and not hasattr(lib, name):
            continue  # an older A/B build (tools/ab_build.sh) without a newer entry point
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPES.get(name, C.c_int)
    _lib = lib
    return lib


def check(status: int):
    if status == HS_OK:
        return
    msg = load().hs_last_error().decode()
    if status == HS_EINVAL:
        raise HoloInvalidArgument(msg)
    if status == HS_ENONFINITE:
        raise HoloNonFinite(msg)
    if status == HS_EOVERFLOW:
        raise HoloOverflow(msg)
    if status == HS_ENOMEM:
        raise MemoryError(msg)
    raise HoloCudaError(msg)

"""ctypes binding of libssg_b200.so (the C ABI in include/ssg_b200.h).

The structures below mirror the header field for field.  Loading fails
loudly: there is no CPU fallback anywhere in this package.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# SSG_B200_LIB selects a diagnostic build of the same library (tools/ only)
LIB_PATH = os.environ.get("SSG_B200_LIB") or os.path.join(_HERE, "libssg_b200.so")

SSG_OK = 0
SSG_ERR_INVALID_ARGUMENT = 1
SSG_ERR_DIM_OVERFLOW = 2
SSG_ERR_CAPACITY = 3
SSG_ERR_CUDA = 4
SSG_PREP_BWD_ACTIVE_ONLY = 1
SSG_BLEND_MAIN_ONLY = 1
SSG_BLEND_EXACT_ONLY = 2
SSG_BLEND_NO_ZERO = 4
SSG_BLEND_ALL_EXACT = 8

EXPORTS = ("ssg_abi_version", "ssg_last_error", "ssg_grid_dims", "ssg_bin_temp_bytes",
           "ssg_preprocess_forward", "ssg_bin_rects", "ssg_bin_prepare", "ssg_bin_finish", "ssg_blend_forward",
           "ssg_blend_backward", "ssg_preprocess_backward", "ssg_blend_backward_slots",
           "ssg_zero_prim_grads", "ssg_preprocess_backward_ex", "ssg_interval_stats_add_ex",
           "ssg_test_sort_temp_bytes",
           "ssg_test_sort", "ssg_test_blend_forward_vanilla", "ssg_adam_step", "ssg_blend_mask_words",
           "ssg_loss_scratch_floats", "ssg_image_loss", "ssg_regularize", "ssg_interval_stats_add",
           "ssg_densify_temp_bytes", "ssg_densify_plan", "ssg_densify_apply", "ssg_ply_unpack",
           "ssg_quantize_u8", "ssg_blend_det_temp_bytes", "ssg_blend_backward_det", "ssg_erf_probe",
           "ssg_pack_splats", "ssg_blend_forward_ex", "ssg_blend_backward_ex",
           "ssg_zero_screen_grads", "ssg_preprocess_forward_views", "ssg_step_value")

_vp = ctypes.c_void_p


class SsgScene(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("sh_degree", ctypes.c_int32),
                ("sh_coeffs", ctypes.c_int32), ("mu", _vp), ("log_scale", _vp), ("rot", _vp),
                ("sh", _vp), ("opacity_logits", _vp), ("beta", _vp), ("dir", _vp)]


class SsgCamera(ctypes.Structure):
    _fields_ = [("R", ctypes.c_double * 9), ("t", ctypes.c_double * 3),
                ("campos", ctypes.c_double * 3), ("fx", ctypes.c_double),
                ("fy", ctypes.c_double), ("cx", ctypes.c_double), ("cy", ctypes.c_double),
                ("tan_fovx", ctypes.c_double), ("tan_fovy", ctypes.c_double),
                ("near_plane", ctypes.c_double), ("s", ctypes.c_double),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32)]


class SsgPrimBuffers(ctypes.Structure):
    _fields_ = [("splat", _vp), ("depth_key", _vp), ("tile_count", _vp), ("tile_rect", _vp),
                ("valid", _vp), ("depth", _vp), ("radius", _vp), ("n_skew_fallback", _vp), ("splat64", _vp)]


class SsgBinBuffers(ctypes.Structure):
    _fields_ = [("depth_order", _vp), ("rank_offset", _vp), ("n_instances", _vp),
                ("capacity", ctypes.c_int64), ("inst_prim", _vp), ("inst_tile", _vp), ("ranges", _vp),
                ("temp", _vp), ("temp_bytes", ctypes.c_size_t)]


class SsgFrameBuffers(ctypes.Structure):
    _fields_ = [("color", _vp), ("final_T", _vp), ("n_contrib", _vp), ("last_idx", _vp), ("blend_mask", _vp),
                ("redo_mask", _vp), ("redo_list", _vp), ("redo_count", _vp)]


class SsgGradBuffers(ctypes.Structure):
    _fields_ = [("screen", _vp), ("d_mu", _vp), ("d_log_scale", _vp), ("d_rot", _vp),
                ("d_sh", _vp), ("d_opacity_logits", _vp), ("d_eta", _vp), ("g_uv", _vp),
                ("g_z", _vp), ("d_beta", _vp)]


class SsgParams(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("sh_degree", ctypes.c_int32), ("sh_coeffs", ctypes.c_int32),
                ("mu", _vp), ("log_scale", _vp), ("rot", _vp), ("sh", _vp), ("opacity_logits", _vp),
                ("beta", _vp), ("dir", _vp)]


class SsgAdamState(ctypes.Structure):
    _fields_ = [(f, _vp) for f in ("m_mu", "v_mu", "m_log_scale", "v_log_scale", "m_rot", "v_rot", "m_sh",
                                   "v_sh", "m_logits", "v_logits", "m_beta", "v_beta", "m_dir", "v_dir",
                                   "row_ok", "n_skipped")]


class SsgDensifyStats(ctypes.Structure):
    _fields_ = [("g_uv", _vp), ("g_z", _vp), ("d_mu", _vp)]


class SsgDensifyCfg(ctypes.Structure):
    _fields_ = [(f, ctypes.c_double) for f in ("tau_uv", "tau_z", "split_scale_threshold", "prune_alpha",
                                               "max_screen_radius", "clone_lr")] + [("max_radii", _vp)]


class SsgAdamHparams(ctypes.Structure):
    _fields_ = [("t", ctypes.c_int64)] + [(f, ctypes.c_double) for f in
                                          ("lr_mu", "lr_scale", "lr_rot", "lr_sh", "lr_opacity", "lr_beta")] + \
               [("skip", _vp)]


SPLAT_BYTES = 64
SPLAT64_BYTES = 64
ABI_VERSION = 7
MAX_BATCH_VIEWS = 8  # SSG_MAX_BATCH_VIEWS

_lib = None


class NativeError(RuntimeError):
    pass


def lib():
    """Load libssg_b200.so; raise if it is missing (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeError(
            f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the sm_100a extension is the only implementation)")
    L = ctypes.CDLL(LIB_PATH)
    L.ssg_last_error.restype = ctypes.c_char_p
    L.ssg_abi_version.restype = ctypes.c_int
    P = ctypes.POINTER
    L.ssg_grid_dims.argtypes = [ctypes.c_int32, ctypes.c_int32, P(ctypes.c_int32), P(ctypes.c_int32)]
    L.ssg_bin_temp_bytes.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                     P(ctypes.c_size_t)]
    L.ssg_preprocess_forward.argtypes = [P(SsgScene), P(SsgCamera), P(SsgPrimBuffers), _vp]
    L.ssg_preprocess_forward_views.argtypes = [P(SsgScene), P(SsgCamera), P(SsgPrimBuffers), ctypes.c_int32, _vp]
    L.ssg_bin_rects.argtypes = [ctypes.c_int64, _vp, _vp, _vp, _vp, ctypes.c_int32,
                                ctypes.c_int32, P(SsgPrimBuffers), _vp]
    L.ssg_bin_prepare.argtypes = [ctypes.c_int64, P(SsgPrimBuffers), P(SsgBinBuffers), _vp]
    L.ssg_bin_finish.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                 P(SsgPrimBuffers), P(SsgBinBuffers), _vp]
    L.ssg_blend_forward.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                    P(ctypes.c_float), _vp, _vp, P(SsgBinBuffers),
                                    P(SsgFrameBuffers), _vp]
    L.ssg_blend_backward.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                     ctypes.c_int32, P(ctypes.c_float), _vp, _vp, P(SsgBinBuffers),
                                     P(SsgFrameBuffers), _vp, P(SsgGradBuffers), _vp]
    L.ssg_blend_forward_ex.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, P(ctypes.c_float), _vp, _vp,
                                       P(SsgBinBuffers), P(SsgFrameBuffers), ctypes.c_int32, _vp]
    L.ssg_blend_backward_ex.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                        P(ctypes.c_float), _vp, _vp, P(SsgBinBuffers), P(SsgFrameBuffers), _vp,
                                        P(SsgGradBuffers), ctypes.c_int32, _vp]
    L.ssg_blend_det_temp_bytes.restype = ctypes.c_size_t
    L.ssg_blend_det_temp_bytes.argtypes = [ctypes.c_int64, ctypes.c_int64]
    L.ssg_blend_backward_det.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                         P(ctypes.c_float), _vp, _vp, P(SsgPrimBuffers), P(SsgBinBuffers),
                                         P(SsgFrameBuffers), _vp, P(SsgGradBuffers), _vp, ctypes.c_size_t, _vp]
    L.ssg_erf_probe.argtypes = [_vp, ctypes.c_int64, _vp, _vp, _vp]
    L.ssg_pack_splats.argtypes = [ctypes.c_int64] + [_vp] * 8
    L.ssg_preprocess_backward.argtypes = [P(SsgScene), P(SsgCamera), P(SsgGradBuffers), _vp]
    L.ssg_zero_prim_grads.argtypes = [ctypes.c_int64, ctypes.c_int32, P(SsgGradBuffers), _vp]
    L.ssg_zero_screen_grads.argtypes = [ctypes.c_int64, P(SsgGradBuffers), _vp]
    L.ssg_preprocess_backward_ex.argtypes = [P(SsgScene), P(SsgCamera), P(SsgGradBuffers), ctypes.c_int32, _vp]
    L.ssg_blend_backward_slots.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                           P(ctypes.c_float), _vp, _vp, P(SsgBinBuffers), P(SsgFrameBuffers),
                                           _vp, _vp, _vp]
    L.ssg_test_blend_forward_vanilla.argtypes = [ctypes.c_int32, ctypes.c_int32, P(ctypes.c_float), _vp, _vp,
                                                 P(SsgBinBuffers), P(SsgFrameBuffers), _vp]
    L.ssg_adam_step.argtypes = [P(SsgParams), P(SsgGradBuffers), P(SsgAdamState), P(SsgAdamHparams), _vp]
    L.ssg_test_sort_temp_bytes.restype = ctypes.c_size_t
    L.ssg_test_sort_temp_bytes.argtypes = [ctypes.c_int64, ctypes.c_int]
    L.ssg_test_sort.argtypes = [_vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int, _vp, _vp]
    L.ssg_ply_unpack.argtypes = [_vp, ctypes.c_int64, ctypes.c_int32, _vp, _vp, ctypes.c_int32, P(SsgParams), _vp]
    L.ssg_quantize_u8.argtypes = [_vp, ctypes.c_int32, ctypes.c_int64, _vp, _vp]
    L.ssg_densify_temp_bytes.restype = ctypes.c_size_t
    L.ssg_densify_temp_bytes.argtypes = [ctypes.c_int64]
    L.ssg_densify_plan.argtypes = [P(SsgScene), P(SsgDensifyStats), P(SsgDensifyCfg), _vp, _vp, ctypes.c_size_t,
                                   P(ctypes.c_int64), P(ctypes.c_double), _vp]
    L.ssg_densify_apply.argtypes = [P(SsgScene), P(SsgParams), _vp, _vp, P(SsgDensifyStats), P(SsgDensifyCfg), _vp,
                                    _vp, _vp, _vp]
    L.ssg_loss_scratch_floats.restype = ctypes.c_int64
    L.ssg_loss_scratch_floats.argtypes = [ctypes.c_int32, ctypes.c_int32]
    L.ssg_image_loss.argtypes = [_vp, _vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_float, _vp, _vp, _vp, _vp]
    L.ssg_step_value.argtypes = [_vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_double, _vp, ctypes.c_int64, _vp, _vp,
                                 _vp]
    L.ssg_regularize.argtypes = [ctypes.c_int64, _vp, _vp, _vp, ctypes.c_float, ctypes.c_float, _vp, _vp, _vp, _vp]
    L.ssg_interval_stats_add.argtypes = [ctypes.c_int64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
    L.ssg_interval_stats_add_ex.argtypes = [ctypes.c_int64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
    L.ssg_blend_mask_words.restype = ctypes.c_int64
    L.ssg_blend_mask_words.argtypes = [ctypes.c_int64, ctypes.c_int32]
    if L.ssg_abi_version() != ABI_VERSION:
        raise NativeError("libssg_b200.so ABI version mismatch; rebuild")
    _lib = L
    return L


def check(status: int, what: str):
    """Map an ssg_status to the reference's exception types."""
    if status == SSG_OK:
        return
    msg = lib().ssg_last_error().decode(errors="replace")
    if status == SSG_ERR_DIM_OVERFLOW:
        raise ValueError("image dimension overflow")
    if status == SSG_ERR_INVALID_ARGUMENT:
        raise ValueError(f"{what}: invalid argument")
    if status == SSG_ERR_CAPACITY:
        raise NativeError(f"{what}: buffer capacity exceeded")
    raise NativeError(f"{what}: CUDA error: {msg}")

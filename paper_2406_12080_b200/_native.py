"""ctypes binding of the C ABI in include/hsplat_b200.h (libhsplat_b200.so).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2406_12080_b200/csrc``).  There is no fallback: if the library
is missing, importing the renderer raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhsplat_b200.so")

u32p = C.POINTER(C.c_uint32)
f32p = C.POINTER(C.c_float)
i32p = C.POINTER(C.c_int32)
u64p = C.POINTER(C.c_uint64)


class hs_camera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("w2c", C.c_float * 12)]


class hs_node_soa(C.Structure):
    _fields_ = [("parent", u32p), ("first_child", u32p), ("child_count", u32p), ("bmin", f32p), ("bmax", f32p),
                ("mean", f32p), ("scale", f32p), ("rot_wxyz", f32p), ("falloff", f32p), ("sh", f32p)]


hs_node_soa_out = hs_node_soa  # identical layout (mutable pointers)


class hs_splat_soa(C.Structure):
    _fields_ = [("mean", f32p), ("scale", f32p), ("rot_wxyz", f32p), ("sh", f32p), ("falloff", f32p),
                ("parent_falloff", f32p), ("t", f32p), ("siblings", i32p)]


hs_splat_soa_out = hs_splat_soa


class hs_grads_out(C.Structure):
    _fields_ = [(k, C.POINTER(C.c_float)) for k in ("mean", "scale", "rot_wxyz", "falloff", "parent_falloff", "t",
                                                    "sh", "mean2d", "exposure")]


class hs_refine_config(C.Structure):
    _fields_ = [("tau_min", C.c_float), ("tau_max", C.c_float), ("steps", C.c_int32), ("lr_mean", C.c_float),
                ("lr_scale", C.c_float), ("lr_rotation", C.c_float), ("lr_falloff", C.c_float),
                ("lr_sh", C.c_float), ("rng_seed", C.c_uint64)]


class hs_gaussian_soa(C.Structure):
    _fields_ = [("mean", f32p), ("scale", f32p), ("rot_wxyz", f32p), ("falloff", f32p), ("sh", f32p)]


hs_gaussian_soa_out = hs_gaussian_soa


class hs_projected(C.Structure):
    """ProjectedSplatT<float> (render.hpp:52-73)."""
    _fields_ = [("culled", C.c_int32), ("mean2d", C.c_float * 2), ("inv_depth", C.c_float),
                ("cam_point", C.c_float * 3), ("cov2d", C.c_float * 4), ("det_pre", C.c_float),
                ("det_post", C.c_float), ("conic", C.c_float * 3), ("alpha_scale", C.c_float),
                ("color", C.c_float * 3), ("color_clamped", C.c_int32 * 3), ("radius", C.c_int32),
                ("tx0", C.c_int32), ("tx1", C.c_int32), ("ty0", C.c_int32), ("ty1", C.c_int32),
                ("falloff_eff", C.c_float), ("parent_falloff_eff", C.c_float), ("falloff_pos", C.c_int32),
                ("parent_falloff_pos", C.c_int32), ("t", C.c_float), ("inv_k", C.c_float)]


class hs_stage_times(C.Structure):
    _fields_ = [("cut_expand", C.c_double), ("weights", C.c_double), ("preprocess", C.c_double),
                ("duplicate", C.c_double), ("tile_ranges", C.c_double), ("alpha_blend", C.c_double)]


class hs_frame_info(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("tiles_x", C.c_int32), ("tiles_y", C.c_int32),
                ("n_splats", C.c_uint64), ("n_visible", C.c_uint64), ("n_duplicates", C.c_uint64),
                ("rendered_count", C.c_int32), ("sort_passes", C.c_int32), ("n_eval", C.c_uint64),
                ("n_contrib", C.c_uint64), ("n_eval_t", C.c_uint64), ("n_exp", C.c_uint64),
                ("n_pow", C.c_uint64), ("n_transition", C.c_uint64)]


HS_OPT_ASYNC = 1
HS_OPT_BLEND_MODE = 2
HS_OPT_DEBUG = 3
HS_OPT_LANES = 4
HS_OPT_STATS = 5

# every symbol include/hsplat_b200.h declares: name -> (restype, argtypes)
_vp = C.c_void_p
_SIGS = {
    "hs_status_name": (C.c_char_p, [C.c_int]),
    "hs_context_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "hs_context_destroy": (None, [_vp]),
    "hs_last_error": (C.c_char_p, [_vp]),
    "hs_context_stream": (_vp, [_vp]),
    "hs_context_synchronize": (C.c_int, [_vp]),
    "hs_context_join": (C.c_int, [_vp]),
    "hs_context_set_option": (C.c_int, [_vp, C.c_int, C.c_int64]),
    "hs_hierarchy_upload": (C.c_int, [_vp, C.POINTER(hs_node_soa), C.c_uint64, C.c_uint32, C.c_int,
                                      C.POINTER(_vp)]),
    "hs_hierarchy_load_h3dg": (C.c_int, [_vp, C.c_char_p, C.POINTER(_vp)]),
    "hs_hierarchy_assemble": (C.c_int, [_vp, C.POINTER(_vp), C.c_uint32, C.POINTER(_vp)]),
    "hs_hierarchy_download": (C.c_int, [_vp, _vp, C.POINTER(hs_node_soa)]),
    "hs_hierarchy_compact": (C.c_int, [_vp, _vp, C.POINTER(hs_camera), C.c_uint64, C.c_float, C.c_float,
                                       C.POINTER(_vp)]),
    "hs_hierarchy_destroy": (None, [_vp]),
    "hs_refine_hierarchy": (C.c_int, [_vp, _vp, C.POINTER(hs_camera), C.POINTER(f32p), f32p, C.c_uint32,
                                      C.POINTER(hs_refine_config), C.POINTER(_vp), C.POINTER(C.c_double), f32p]),
    "hs_photometric_loss": (C.c_int, [_vp, f32p, f32p, C.c_int32, C.c_int32, f32p, f32p]),
    "hs_hierarchy_node_count": (C.c_uint64, [_vp]),
    "hs_hierarchy_leaf_count": (C.c_uint64, [_vp]),
    "hs_cut_create": (C.c_int, [_vp, C.POINTER(_vp)]),
    "hs_cut_destroy": (None, [_vp]),
    "hs_select_cut": (C.c_int, [_vp, _vp, C.POINTER(hs_camera), C.c_float, _vp]),
    "hs_cut_size": (C.c_int, [_vp, _vp, u64p]),
    "hs_cut_download": (C.c_int, [_vp, _vp, u32p, f32p, f32p]),
    "hs_cut_upload": (C.c_int, [_vp, _vp, u32p, f32p, f32p, C.c_uint64, _vp]),
    "hs_cut_render_splats": (C.c_int, [_vp, _vp, _vp, C.POINTER(hs_splat_soa)]),
    "hs_transfer_tracker_create": (C.c_int, [_vp, _vp, C.POINTER(_vp)]),
    "hs_transfer_tracker_destroy": (None, [_vp]),
    "hs_transfer_count": (C.c_int, [_vp, _vp, _vp, u64p]),
    "hs_frame_create": (C.c_int, [_vp, C.POINTER(_vp)]),
    "hs_frame_destroy": (None, [_vp]),
    "hs_render_hierarchy": (C.c_int, [_vp, _vp, C.POINTER(hs_camera), C.c_float, _vp, _vp,
                                      C.POINTER(hs_stage_times)]),
    "hs_render_cut": (C.c_int, [_vp, _vp, _vp, C.POINTER(hs_camera), _vp, C.POINTER(hs_stage_times)]),
    "hs_render_splats": (C.c_int, [_vp, C.POINTER(hs_splat_soa), C.c_uint64, C.POINTER(hs_camera), _vp,
                                   C.POINTER(hs_stage_times)]),
    "hs_render_backward": (C.c_int, [_vp, _vp, f32p, f32p, f32p, C.POINTER(hs_grads_out)]),
    "hs_frame_wait": (C.c_int, [_vp, _vp]),
    "hs_frame_get_info": (C.c_int, [_vp, _vp, C.POINTER(hs_frame_info)]),
    "hs_frame_download": (C.c_int, [_vp, _vp, f32p, f32p, f32p, i32p]),
    "hs_frame_download_async": (C.c_int, [_vp, _vp, f32p, f32p, f32p]),
    "hs_frame_download_wait": (C.c_int, [_vp, _vp, i32p]),
    "hs_frame_download_device": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "hs_kernel_launch_count": (C.c_uint64, []),
    "hs_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(_vp)]),
    "hs_host_free": (None, [_vp]),
    "hs_frame_debug":(C.c_int, [_vp, _vp, u64p, u64p, u32p, u64p, u32p, f32p]),
    "hs_synth_node_count": (C.c_uint64, [C.c_uint64]),
    "hs_synth_scene_side": (C.c_float, [C.c_uint64]),
    "hs_synth_city": (C.c_int, [C.c_uint64, C.c_uint64, C.c_int, C.POINTER(hs_node_soa)]),
    "hs_synth_city_chunk": (C.c_int, [C.c_uint64, C.c_uint64, C.c_float, C.c_float, C.c_int,
                                      C.POINTER(hs_node_soa)]),
    "hs_synth_skybox": (C.c_int, [C.c_uint64, C.c_float, C.c_uint64, C.POINTER(C.c_float), C.c_int,
                                  C.POINTER(hs_node_soa)]),
    "hs_build_bvh": (C.c_int, [f32p, f32p, f32p, f32p, f32p, C.c_uint64, C.c_int, C.POINTER(hs_node_soa)]),
    "hs_h3dg_read_header":(C.c_int, [C.c_char_p, u64p, C.POINTER(C.c_uint32)]),
    "hs_h3dg_read": (C.c_int, [C.c_char_p, C.POINTER(hs_node_soa), C.c_uint64]),
    "hs_h3dg_write": (C.c_int, [C.c_char_p, C.POINTER(hs_node_soa), C.c_uint64, C.c_uint32]),
    "hs_validate_hierarchy": (C.c_int, [C.POINTER(hs_node_soa), C.c_uint64, C.c_char_p, C.c_size_t]),
    "hs_granularity": (C.c_int, [_vp, f32p, f32p, C.c_uint64, C.POINTER(hs_camera), f32p]),
    "hs_interp_weight": (C.c_int, [_vp, f32p, f32p, C.c_uint64, C.c_float, f32p]),
    "hs_transition_alpha": (C.c_int, [_vp, f32p, i32p, C.c_uint64, f32p]),
    "hs_interpolated_gaussians": (C.c_int, [_vp, C.POINTER(hs_gaussian_soa), C.POINTER(hs_gaussian_soa), f32p, i32p,
                                            C.c_uint64, C.POINTER(hs_gaussian_soa)]),
    "hs_assemble_cut_splats": (C.c_int, [_vp, _vp, C.POINTER(hs_gaussian_soa), C.c_uint64, u32p, f32p, C.c_uint64,
                                         C.POINTER(hs_splat_soa)]),
    "hs_project": (C.c_int, [_vp, C.POINTER(hs_splat_soa), C.c_uint64, C.POINTER(hs_camera),
                             C.POINTER(hs_projected)]),
    "hs_render_reference": (C.c_int, [_vp, C.POINTER(hs_splat_soa), C.c_uint64, C.POINTER(hs_camera), _vp]),
    "hs_frame_order": (C.c_int, [_vp, _vp, u32p, u64p]),
    "hs_read_cameras": (C.c_int, [C.c_char_p, C.POINTER(hs_camera), C.c_uint64, u64p, C.c_char_p, C.c_size_t]),
    "hs_read_camera_path": (C.c_int, [C.c_char_p, C.POINTER(C.c_double), C.POINTER(hs_camera), C.c_uint64, u64p,
                                      C.c_char_p, C.c_size_t]),
    "hs_write_cameras": (C.c_int, [C.c_char_p, C.POINTER(hs_camera), C.c_uint64, C.c_char_p, C.c_size_t]),
    "hs_write_camera_path": (C.c_int, [C.c_char_p, C.POINTER(C.c_double), C.POINTER(hs_camera), C.c_uint64,
                                       C.c_char_p, C.c_size_t]),
}

_lib = None


def lib():
    """Load libhsplat_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (the CUDA path has no fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def ptr(a: np.ndarray | None, ctype):
    if a is None:
        return C.cast(None, C.POINTER(ctype))
    assert a.flags["C_CONTIGUOUS"], "arrays passed to the C ABI must be contiguous"
    return a.ctypes.data_as(C.POINTER(ctype))

"""ctypes binding of ``libdeformtrack_b200.so`` (include/deformtrack_b200.h).

The library is the product: there is no CPU fallback. Importing this module on a host
without the built library raises; calling into it without a CUDA device raises from
the first CUDA call. Device memory on the Python side is held in torch tensors, whose
raw pointers cross the C-ABI (torch is plumbing here, not compute).
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from . import exceptions as exc

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("DEFORMTRACK_B200_LIB", _PKG / "libdeformtrack_b200.so"))

DT_OK = 0
DT_ERR_INVALID_ARGUMENT = 1
DT_ERR_CUDA = 2
DT_ERR_NO_VALID_HYPOTHESIS = 3
DT_ERR_EMPTY_TEMPLATE = 4
DT_ERR_ALL_ZERO_WEIGHTS = 5
DT_ERR_UNSUPPORTED = 6
DT_ERR_NOT_BOUND = 7

P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int32
F64 = C.c_double


class PreselectParams(C.Structure):
    _fields_ = [
        ("distance_threshold", F64),
        ("n_reweight_iters", I32),
        ("inlier_weight_min", F64),
        ("min_support", F64),
    ]


class Config(C.Structure):
    _fields_ = [
        ("feature_weight", F64), ("arap_weight", F64), ("angle_weight", F64),
        ("rotation_weight", F64), ("tukey_scale", F64), ("data_floor", F64),
        ("max_outer_iters", I32),
        ("lambda_init", F64), ("lambda_decrease", F64), ("lambda_increase", F64),
        ("lambda_min", F64), ("lambda_max", F64),
        ("max_retries", I32),
        ("step_tol", F64), ("cost_tol", F64), ("gate_distance", F64), ("cos_gate", F64),
        ("preselect", PreselectParams),
        ("fx", F64), ("fy", F64), ("cx", F64), ("cy", F64),
        ("width", I32), ("height", I32),
        ("z_min", F64), ("z_max", F64),
        ("sampling_radius", F64),
        ("cluster_size", I32),
        ("max_hamming", I32),
    ]


class Report(C.Structure):
    _fields_ = [
        ("icp_cost", F64), ("feature_cost", F64), ("arap_cost", F64), ("total_cost", F64),
        ("match_weight_sum", F64), ("final_step_norm", F64), ("preselect_support", F64),
        ("n_correspondences", I32), ("n_matches", I32), ("n_preselected", I32),
        ("outer_iterations", I32), ("accepted_steps", I32), ("rejected_steps", I32),
        ("stalled", I32), ("converged", I32), ("n_cost_history", I32),
        ("preselect_status", I32), ("preselect_reference", I32), ("frame_id", I32),
    ]


class FrameInput(C.Structure):
    _fields_ = [
        ("depth", P), ("normals", P), ("match_src", P), ("match_dst", P), ("match_w", P),
        ("match_bidx", P), ("match_bw", P), ("n_pairs", I64),
        ("frame_desc", P), ("frame_kp", P), ("n_frame", I64), ("refs", P), ("n_refs", I64),
        ("use_matches", I32), ("on_device", I32), ("frame_id", I32),
        ("height", I32), ("width", I32), ("depth_kind", I32),
    ]


class FrameOutput(C.Structure):
    _fields_ = [
        ("warps", P), ("points", P), ("normals", P), ("match_weights", P), ("match_flags", P),
        ("match_src", P), ("match_dst", P), ("match_capacity", I64),
        ("control_data_weights", P), ("report", P),
        ("cost_history", P), ("lambda_history", P), ("stalled", P),
    ]


# name -> argtypes (restype is int status unless noted)
_SIGNATURES: dict[str, list] = {
    "dt_device_info": [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)],
    "dt_observation_normals": [P, I64, I64, F64, F64, F64, F64, F64, F64, P, P, P],
    "dt_warp_and_rasterize": [P, P, P, P, I64, I64, P, I64, P, P, P, I64, I64, F64, F64, F64, F64,
                              F64, F64, P, P, P, P, P, P, P],
    "dt_icp_reduce": [P, P, P, P, P, I64, I64, P, P, I64, F64, P, C.c_int, C.c_int, P, P, P, P, P],
    "dt_feature_reduce": [P, P, P, P, P, I64, I64, P, P, I64, F64, C.c_int, P, P, P, P],
    "dt_arap_reduce": [P, P, P, P, P, P, I64, P, I64, F64, F64, C.c_int, P, P, P],
    "dt_solve_damped": [P, P, P, I64, P, P, P],
    "dt_apply_step": [P, P, I64, P, P],
    "dt_warp_increment_basis": [P, I64, P, P],
    "dt_dq_to_transform": [P, I64, P, P, P],
    "dt_warp_all": [P, P, P, P, I64, I64, P, P, P, P],
    "dt_bind_points": [P, I64, P, I64, I64, F64, P, P, P],
    "dt_hamming_match": [P, I64, P, I64, P, P, P],
    "dt_preselect": [P, P, I64, P, I64, C.POINTER(PreselectParams), P, P, P, P, P, P, P],
    "dt_sample_control_points": [P, I64, F64, P, P, C.c_int],
    "dt_connection_candidates": [P, I64, F64, P, P, I64, P, C.c_int],
    "dt_build_connections": [P, I64, F64, F64, P, P, I64, P, C.c_int],
    "dt_estimate_point_normals": [P, I64, I64, P, C.c_int],
    "dt_orb_create": [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, P, P, C.c_int,
                      C.POINTER(P)],
    "dt_orb_destroy": [P],
    "dt_orb_detect": [P, P, C.c_int, P, P, P, P, P],
    "dt_orb_last": [P, C.POINTER(P), C.POINTER(P), P],
    "dt_tracker_create": [C.POINTER(Config), P, P, P, P, I64, I64, P, P, I64, P, P, I64, C.c_int,
                          P, C.POINTER(P)],
    "dt_tracker_destroy": [P],
    "dt_tracker_set_features": [P, P, P, I64, P, P],
    "dt_tracker_set_warps": [P, P, C.c_int],
    "dt_tracker_get_warps": [P, P],
    "dt_tracker_set_config": [P, C.POINTER(Config)],
    "dt_tracker_sync": [P],
    "dt_track_frame": [P, C.POINTER(FrameInput), C.POINTER(FrameOutput)],
    "dt_tracker_get_history": [P, P, P, P],
    "dt_tracker_device_outputs": [P, C.POINTER(P), C.POINTER(P), C.POINTER(P)],
    "dt_tracker_last_launches": [P],
    "dt_track_frames_batched": [C.POINTER(P), C.POINTER(FrameInput), C.POINTER(FrameOutput),
                                I32, P],
    "dt_track_frame_async": [P, C.POINTER(FrameInput)],
    "dt_tracker_collect": [P, C.POINTER(FrameInput), C.POINTER(FrameOutput)],
    "dt_track_frame_submit": [P, C.POINTER(FrameInput), C.POINTER(FrameOutput)],
    "dt_tracker_wait": [P],
    "dt_tracker_set_profiling": [P, C.c_int],
    "dt_tracker_get_phase_ms": [P, P],
    "dt_tracker_get_trace": [P, P, C.c_int],
    "dt_tracker_get_arrivals": [P, P, C.c_int],
    "dt_depth_from_pfm": [P, I64, I64, C.c_int, P, P],
    "dt_stereo_create": [C.c_int, C.c_int, C.c_int, C.c_int, F64, F64, F64, C.c_int, C.c_int,
                         C.POINTER(P)],
    "dt_stereo_destroy": [P],
    "dt_stereo_compute": [P, P, P, C.c_int, P, P, P],
    "dt_stereo_last": [P, C.POINTER(P)],
}

# int64-returning codecs (host memory; no device needed)
_SIGNATURES_I64: dict[str, list] = {
    "dt_format_reals": [P, I64, I64, P, I64],
    "dt_parse_reals": [P, I64, P, I64],
}

N_PHASES = 6
PHASES = ("normals", "orb_match", "preselect", "match_prep", "lm_solver", "warp_out")

EXPORTED = ["dt_last_error", "dt_version", "dt_tracker_stream", *_SIGNATURES, *_SIGNATURES_I64]

DT_DEPTH_F64 = 0
DT_DEPTH_PFM = 1


def _require_built() -> None:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build the sm_100a library first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback"
        )


def _load() -> C.CDLL:
    _require_built()
    lib = C.CDLL(str(LIB_PATH))
    lib.dt_last_error.restype = C.c_char_p
    lib.dt_last_error.argtypes = []
    lib.dt_version.restype = C.c_char_p
    lib.dt_version.argtypes = []
    for name, argtypes in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = C.c_int
    for name, argtypes in _SIGNATURES_I64.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = I64
    lib.dt_tracker_stream.argtypes = [P]
    lib.dt_tracker_stream.restype = P
    return lib


class _Lib:
    """The library handle, opened (dlopen) at the first call into it. Importing the
    package only checks that the library is built (and raises ImportError if not), so
    the host-only pieces -- config objects, the synthetic scene generator, the oracle
    arm of bench.py -- never map the CUDA library into a process that does no device
    work."""

    _cdll: C.CDLL | None = None

    def __getattr__(self, name: str):
        if _Lib._cdll is None:
            _Lib._cdll = _load()
        fn = getattr(_Lib._cdll, name)
        setattr(self, name, fn)
        return fn


_require_built()
lib = _Lib()


def loaded() -> bool:
    """Whether the CUDA library has been mapped into this process."""
    return _Lib._cdll is not None


def check(status: int, what: str = "") -> None:
    """Raise the exception class mirroring the reference's for a non-zero status."""
    if status == DT_OK:
        return
    msg = lib.dt_last_error().decode(errors="replace")
    label = f"{what}: {msg}" if what else msg
    if status == DT_ERR_INVALID_ARGUMENT:
        raise ValueError(label)
    if status == DT_ERR_NO_VALID_HYPOTHESIS:
        raise exc.NoValidHypothesis(label)
    if status == DT_ERR_EMPTY_TEMPLATE:
        raise exc.EmptyTemplate(label)
    if status == DT_ERR_ALL_ZERO_WEIGHTS:
        raise exc.AllZeroWeights(label)
    if status == DT_ERR_NOT_BOUND:
        raise ValueError(label)
    if status == DT_ERR_UNSUPPORTED:
        raise NotImplementedError(label)
    raise RuntimeError(f"CUDA error in deformtrack_b200 ({label})")


def version() -> str:
    return lib.dt_version().decode()

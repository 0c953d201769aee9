"""ctypes binding of the C ABI in include/b200geo.h (libb200geo.so, built in-tree).

The product path: there is no CPU fallback. Importing this module on a machine
where the library is missing raises immediately; calls that need a GPU fail
loudly through the library's own CUDA error reporting.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libb200geo.so")

DG_OK, DG_EINVAL, DG_ERUNTIME, DG_ENOMEM = 0, 1, 2, 3


class dg_pair_offsets(C.Structure):
    _fields_ = [("tdoa_samples", C.c_int64), ("fdoa_hz", C.c_double)]


class dg_ecef(C.Structure):
    _fields_ = [("x", C.c_double), ("y", C.c_double), ("z", C.c_double)]


class dg_state(C.Structure):
    _fields_ = [("position", dg_ecef), ("velocity", dg_ecef)]


class dg_latlon_bounds(C.Structure):
    _fields_ = [("lat_min_deg", C.c_double), ("lat_max_deg", C.c_double),
                ("lon_min_deg", C.c_double), ("lon_max_deg", C.c_double)]


class dg_emitter_estimate(C.Structure):
    _fields_ = [("lat_deg", C.c_double), ("lon_deg", C.c_double), ("alt_m", C.c_double),
                ("grid_index", C.c_int64), ("score", C.c_double), ("score_zsigma", C.c_double)]


class dg_snapshots(C.Structure):
    _fields_ = [("n_snapshots", C.c_int64), ("n_receivers", C.c_int64), ("n_samples", C.c_int64),
                ("sample_rate_hz", C.c_double), ("center_freq_hz", C.c_double),
                ("states", C.POINTER(dg_state)),
                ("captures_iq", C.POINTER(C.POINTER(C.c_double))),
                ("captures_f32", C.POINTER(C.POINTER(C.c_float)))]


class dg_iq_header(C.Structure):
    _fields_ = [("sample_rate_hz", C.c_double), ("center_freq_hz", C.c_double),
                ("start_time_s", C.c_double), ("sample_count", C.c_int64)]


class dg_grid_axes(C.Structure):
    _fields_ = [("lat_start_deg", C.c_double), ("lat_step_deg", C.c_double),
                ("lat_count", C.c_int64), ("lon_start_deg", C.c_double),
                ("lon_step_deg", C.c_double), ("lon_count", C.c_int64),
                ("altitude_m", C.c_double)]


class dg_emitter_def(C.Structure):
    _fields_ = [("lat_deg", C.c_double), ("lon_deg", C.c_double), ("alt_m", C.c_double),
                ("waveform", C.c_int), ("prn", C.c_int), ("data_seed", C.c_uint64),
                ("tone_offset_hz", C.c_double), ("bandwidth_hz", C.c_double),
                ("period_s", C.c_double), ("ref_snr_db", C.c_double), ("ref_range_m", C.c_double)]


class dg_receiver_def(C.Structure):
    _fields_ = [("alt_m", C.c_double), ("inclination_deg", C.c_double), ("raan_deg", C.c_double),
                ("phase_deg", C.c_double), ("states", C.POINTER(dg_state))]


class dg_scenario(C.Structure):
    _fields_ = [("receivers", C.POINTER(dg_receiver_def)), ("n_receivers", C.c_int64),
                ("emitters", C.POINTER(dg_emitter_def)), ("n_emitters", C.c_int64),
                ("snapshot_count", C.c_int64), ("snapshot_spacing_s", C.c_double),
                ("capture_duration_s", C.c_double), ("sample_rate_hz", C.c_double),
                ("center_freq_hz", C.c_double), ("start_time_s", C.c_double),
                ("noise_seed", C.c_uint64), ("noise_power", C.c_double)]


class dg_options(C.Structure):
    _fields_ = [("k_sigma", C.c_double), ("exclusion_radius_cells", C.c_int),
                ("normalize_per_snapshot", C.c_int), ("detect", C.c_int),
                ("stream", C.c_void_p), ("profile", C.c_int), ("patch_peak", C.c_int),
                ("peak_stage", C.c_int), ("peak_max", C.c_double)]


class dg_work_unit(C.Structure):
    _fields_ = [("step", C.c_int64), ("part", C.c_int32), ("parts", C.c_int32),
                ("rank", C.c_int32), ("reserved", C.c_int32)]


class dg_tuning(C.Structure):
    _fields_ = [("correlator", C.c_int), ("moment_block", C.c_int), ("moment_count", C.c_int),
                ("evaluate_tensor", C.c_int), ("refine_tau", C.c_double),
                ("allow_weaker_refine", C.c_int), ("direct_refine_tau", C.c_double),
                ("noise_refine_tau", C.c_double), ("surface_budget_bytes", C.c_int64),
                ("moment_fft", C.c_int), ("fft_refine_kappa", C.c_double)]


DG_CORRELATOR_AUTO, DG_CORRELATOR_DIRECT, DG_CORRELATOR_MOMENTS = 0, 1, 2


class dg_result(C.Structure):
    _fields_ = [("accumulated", C.POINTER(C.c_double)),
                ("accumulated_device", C.c_void_p),
                ("per_snapshot", C.POINTER(C.c_double)),
                ("detections", C.POINTER(dg_emitter_estimate)),
                ("detections_capacity", C.c_int64),
                ("n_detections", C.c_int64),
                ("argmax_index", C.c_int64),
                ("argmax_value", C.c_double),
                ("n_refined", C.c_int64),
                ("n_reranked", C.c_int64),
                ("sum_overlap_samples", C.c_double),
                ("correlate_ms", C.c_double),
                ("correlate_launches", C.c_int64),
                ("total_ms", C.c_double),
                ("kernel_launches", C.c_int64),
                ("moments_ms", C.c_double),
                ("evaluate_ms", C.c_double),
                ("moment_ffma2", C.c_double),
                ("evaluate_ffma2", C.c_double),
                ("direct_steps", C.c_int64),
                ("evaluate_tc_flop", C.c_double),
                ("moment_fft_flop", C.c_double)]


# every symbol include/b200geo.h declares (tests check the .so exports them)
EXPORTS = (
    "dg_last_error", "dg_abi_version", "dg_engine_create", "dg_engine_destroy",
    "dg_device_count", "dg_engine_create_multi",
    "dg_engine_descriptor", "dg_stage", "dg_stage_f32", "dg_session_destroy",
    "dg_correlate_batch", "dg_build_candidate_grid", "dg_grid_slab", "dg_grid_from_points",
    "dg_grid_info", "dg_grid_points", "dg_grid_destroy", "dg_predict_offsets",
    "dg_correlate_snapshot", "dg_options_default", "dg_geolocate_snapshots",
    "dg_stage_snapshots", "dg_geolocate_staged", "dg_staged_destroy", "dg_correlate_steps",
    "dg_accumulate_peak", "dg_detect_emitters", "dg_read_iq_header", "dg_read_iq",
    "dg_stage_snapshots_iq", "dg_write_grid", "dg_render_heatmap", "dg_write_detections_csv",
    "dg_read_grid", "dg_grid_from_axes", "dg_format_g17", "dg_scenario_samples",
    "dg_simulate_scenario",
    "dg_tuning_default", "dg_engine_set_tuning", "dg_engine_get_tuning", "dg_shard_plan",
    "dg_correlate_units",
    "dg_plan_batches", "dg_fp32_peak_tflops", "dg_fp32x2_peak_tflops", "dg_fp64_peak_tflops",
)

_vp = C.c_void_p
_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the B200 engine has no CPU fallback. Build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (nvcc, sm_100a).")
    L = C.CDLL(LIB_PATH)
    L.dg_last_error.restype = C.c_char_p
    L.dg_abi_version.restype = C.c_int
    sigs = {
        "dg_engine_create": [C.c_int, C.POINTER(_vp)],
        "dg_engine_create_multi": [C.POINTER(C.c_int), C.c_int, C.POINTER(_vp)],
        "dg_device_count": [C.POINTER(C.c_int)],
        "dg_engine_descriptor": [_vp, C.c_char_p, C.c_size_t, C.c_char_p, C.c_size_t,
                                 C.POINTER(C.c_uint)],
        "dg_stage": [_vp, _dp, C.c_int64, C.c_double, _dp, C.c_int64, C.c_double, C.POINTER(_vp)],
        "dg_stage_f32": [_vp, C.POINTER(C.c_float), C.c_int64, C.c_double,
                         C.POINTER(C.c_float), C.c_int64, C.c_double, C.POINTER(_vp)],
        "dg_correlate_batch": [_vp, C.POINTER(dg_pair_offsets), C.c_int64, _dp, C.c_int64],
        "dg_build_candidate_grid": [_vp, C.POINTER(dg_latlon_bounds), C.c_double, C.c_double,
                                    C.c_uint64, C.POINTER(_vp)],
        "dg_grid_slab": [_vp, C.c_int64, C.c_int64, C.POINTER(_vp)],
        "dg_grid_from_points": [_vp, C.POINTER(dg_ecef), C.c_int64, C.c_double, C.c_double,
                                C.c_int64, C.c_double, C.c_double, C.c_int64, C.c_double,
                                C.POINTER(_vp)],
        "dg_grid_info": [_vp, _dp, _dp, _i64p, _dp, _dp, _i64p, _dp, _i64p],
        "dg_grid_points": [_vp, C.POINTER(dg_ecef)],
        "dg_predict_offsets": [_vp, _vp, C.POINTER(dg_state), C.POINTER(dg_state), C.c_double,
                               C.c_double, C.POINTER(dg_pair_offsets)],
        "dg_correlate_snapshot": [_vp, _vp, C.POINTER(dg_state), C.POINTER(dg_state),
                                  C.c_double, _dp],
        "dg_geolocate_snapshots": [_vp, _vp, C.POINTER(dg_snapshots), C.POINTER(dg_options),
                                   C.POINTER(dg_result)],
        "dg_stage_snapshots": [_vp, C.POINTER(dg_snapshots), C.POINTER(_vp)],
        "dg_geolocate_staged": [_vp, _vp, _vp, C.POINTER(dg_options), C.POINTER(dg_result)],
        "dg_correlate_steps": [_vp, _vp, _vp, C.c_int64, C.c_int64, C.POINTER(dg_options), _vp,
                               _vp, C.POINTER(dg_result)],
        "dg_accumulate_peak": [_vp, _vp, _vp, _vp, _vp, C.POINTER(dg_options),
                               C.POINTER(dg_result)],
        "dg_detect_emitters": [_vp, _vp, _vp, C.c_int, C.c_double, C.c_int,
                               C.POINTER(dg_emitter_estimate), C.c_int64, _i64p],
        "dg_read_iq_header": [C.c_char_p, C.POINTER(dg_iq_header)],
        "dg_read_iq": [C.c_char_p, C.POINTER(dg_iq_header), C.POINTER(C.c_float), C.c_int64],
        "dg_stage_snapshots_iq": [_vp, C.POINTER(C.c_char_p), C.c_int64, C.c_int64,
                                  C.POINTER(dg_state), C.POINTER(_vp)],
        "dg_write_grid": [_vp, _vp, _vp, C.c_int, C.c_char_p, C.c_int],
        "dg_render_heatmap": [_vp, _vp, _vp, C.c_int, C.c_char_p],
        "dg_write_detections_csv": [C.POINTER(dg_emitter_estimate), C.c_int64, C.c_char_p],
        "dg_read_grid": [C.c_char_p, C.POINTER(dg_grid_axes), _dp, C.c_int64],
        "dg_grid_from_axes": [_vp, C.POINTER(dg_grid_axes), C.POINTER(_vp)],
        "dg_format_g17": [_vp, _dp, C.c_int64, C.c_char_p, C.POINTER(C.c_uint8)],
        "dg_scenario_samples": [C.POINTER(dg_scenario), _i64p],
        "dg_simulate_scenario": [_vp, C.POINTER(dg_scenario), C.POINTER(_vp), _dp,
                                 C.POINTER(dg_state), _dp],
        "dg_shard_plan": [C.c_int64, C.c_int64, C.c_int, C.c_int, C.POINTER(dg_work_unit),
                          C.c_int64, _i64p],
        "dg_correlate_units": [_vp, _vp, _vp, C.POINTER(dg_work_unit), C.c_int64,
                               C.POINTER(dg_options), _vp, C.POINTER(dg_result)],
        "dg_engine_set_tuning": [_vp, C.POINTER(dg_tuning)],
        "dg_engine_get_tuning": [_vp, C.POINTER(dg_tuning)],
        "dg_fp32_peak_tflops": [C.c_int, _dp],
        "dg_fp32x2_peak_tflops": [C.c_int, _dp],
        "dg_fp64_peak_tflops": [C.c_int, _dp],
        "dg_plan_batches": [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                            C.POINTER(C.c_uint64)],
    }
    for name, args in sigs.items():
        fn = getattr(L, name)
        fn.restype = C.c_int
        fn.argtypes = args
    for name in ("dg_engine_destroy", "dg_session_destroy", "dg_grid_destroy",
                 "dg_staged_destroy"):
        fn = getattr(L, name)
        fn.restype = None
        fn.argtypes = [_vp]
    L.dg_tuning_default.restype = None
    L.dg_tuning_default.argtypes = [C.POINTER(dg_tuning)]
    L.dg_options_default.restype = None
    L.dg_options_default.argtypes = [C.POINTER(dg_options)]
    return L


lib = _load()


def check(rc: int) -> None:
    """Raise the reference's exception type for a C ABI error code."""
    if rc == DG_OK:
        return
    msg = lib.dg_last_error().decode()
    if rc == DG_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if rc == DG_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)  # std::runtime_error

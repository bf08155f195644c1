"""ctypes declarations for include/zsim_gpu.h and the loader of libzsim_gpu.so.

The product path has no CPU fallback: if the native library is missing this
module raises at import time.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("ZSIM_GPU_LIB", _PKG / "libzsim_gpu.so"))

c_double_p = C.POINTER(C.c_double)
c_float_p = C.POINTER(C.c_float)
c_int32_p = C.POINTER(C.c_int32)
c_uint8_p = C.POINTER(C.c_uint8)
c_uint64_p = C.POINTER(C.c_uint64)


class SimConfigC(C.Structure):
    _fields_ = [
        ("wheelbase", C.c_double), ("ego_length", C.c_double), ("ego_width", C.c_double),
        ("ego_center_offset", C.c_double), ("delta_max", C.c_double), ("v_min", C.c_double),
        ("goal_radius", C.c_double), ("footprint_margin", C.c_double), ("stop_cross_speed", C.c_double),
        ("stop_zone", C.c_double), ("stop_slow_speed", C.c_double), ("disable_dones", C.c_int32),
        ("n_agents", C.c_int32), ("n_road", C.c_int32), ("n_route", C.c_int32),
        ("w_progress", C.c_double), ("w_speed", C.c_double), ("w_lat", C.c_double), ("w_lon", C.c_double),
        ("terminal_penalty", C.c_double), ("feature_radius", C.c_double), ("threads", C.c_int32),
        ("reserved", C.c_int32),
    ]


class StateView(C.Structure):
    _fields_ = [
        ("x", c_double_p), ("y", c_double_p), ("heading", c_double_p), ("v", c_double_p),
        ("steering", c_double_p), ("t", c_int32_p), ("done", c_uint8_p), ("reason", c_uint8_p),
        ("rng", c_uint64_p), ("proj_s", c_double_p), ("proj_d", c_double_p), ("proj_in_corridor", c_uint8_p),
        ("events", c_uint8_p), ("stopped_flags", c_uint8_p),
    ]


class StepOutView(C.Structure):
    _fields_ = [("reward", c_float_p), ("event", c_uint8_p), ("s", c_float_p), ("a_lat", c_float_p),
                ("a_lon", c_float_p), ("v", c_float_p)]


class ObsView(C.Structure):
    _fields_ = [("active", c_float_p), ("agents", c_float_p), ("road", c_float_p), ("route", c_float_p),
                ("value_only", c_float_p)]


class ModelConfigC(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("latent", "heads", "trunk_blocks", "value_embed", "n_agents", "n_road",
                                          "n_route", "n_accel", "n_steer", "reserved")]


class EnvInfo(C.Structure):
    _fields_ = [
        ("batch", C.c_int32), ("horizon", C.c_int32), ("dt", C.c_double), ("total_stop_lines", C.c_int32),
        ("zero_accel_idx", C.c_int32), ("zero_steer_idx", C.c_int32), ("num_accel", C.c_int32),
        ("num_steer", C.c_int32), ("cap_steps", C.c_int32), ("cap_agents", C.c_int32), ("cap_road", C.c_int32),
        ("cap_route", C.c_int32), ("cap_lanes", C.c_int32), ("cap_vertices", C.c_int32),
        ("cap_lights", C.c_int32), ("cap_stops", C.c_int32), ("device", C.c_int32),
        ("static_bytes", C.c_uint64), ("scenarios", C.c_int32), ("controlled", C.c_int32),
        ("step_observe_kernels", C.c_int32), ("reserved0", C.c_int32),
    ]


class EpisodeView(C.Structure):
    _fields_ = [("accel_idx", c_int32_p), ("steer_idx", c_int32_p), ("logp", c_float_p), ("value", c_float_p),
                ("reward", c_float_p), ("s", c_float_p), ("a_lat", c_float_p), ("a_lon", c_float_p),
                ("v", c_float_p), ("done", c_uint8_p), ("mask", c_uint8_p), ("bootstrap", c_float_p),
                ("terminal", c_uint8_p), ("events", c_uint8_p), ("initial_s", c_float_p),
                ("logged_progress", c_float_p), ("horizon", C.c_int32), ("reserved", C.c_int32)]


class SequencesView(C.Structure):
    _fields_ = [("capacity", C.c_int32), ("seq_len", C.c_int32), ("obs", ObsView), ("accel_idx", c_int32_p),
                ("steer_idx", c_int32_p), ("logmu", c_float_p), ("reward", c_float_p), ("done", c_uint8_p),
                ("mask", c_uint8_p), ("bootstrap", c_float_p), ("row", c_int32_p), ("t0", c_int32_p),
                ("count", c_int32_p)]


class ScoreBounds(C.Structure):
    _fields_ = [("progress", C.c_double), ("collision", C.c_double), ("off_route", C.c_double),
                ("stop_line", C.c_double), ("traffic_light", C.c_double), ("comfort", C.c_double)]


class ComfortWeights(C.Structure):
    _fields_ = [("w_accel", C.c_double), ("w_jerk", C.c_double)]


class MetricView(C.Structure):
    _fields_ = [(n, c_double_p) for n in ("relative_progress_raw", "relative_progress", "collision_free",
                                          "off_route_free", "stop_line_free", "traffic_light_free",
                                          "mixed_comfort", "scenario_score")] + \
               [(n, c_uint8_p) for n in ("degenerate", "failed", "goal_reached")]


class StressConfigC(C.Structure):
    _fields_ = [("count", C.c_int32), ("num_steps", C.c_int32), ("agents", C.c_int32),
                ("road_points", C.c_int32), ("lanes", C.c_int32), ("lane_vertices", C.c_int32),
                ("dt", C.c_double), ("speed_limit", C.c_double), ("lane_width", C.c_double),
                ("first_index", C.c_int32), ("flags", C.c_int32)]


# name -> (restype, argtypes); every symbol include/zsim_gpu.h declares.
_P = C.c_void_p
SIGNATURES = {
    "zsim_abi_version": (C.c_int, []),
    "zsim_last_error": (C.c_char_p, []),
    "zsim_sim_config_defaults": (C.c_int, [C.POINTER(SimConfigC)]),
    "zsim_env_create": (C.c_int, [_P, C.c_size_t, C.POINTER(C.c_int64), C.c_int32, C.c_int32,
                                  C.POINTER(SimConfigC), c_double_p, C.c_int32, c_double_p, C.c_int32,
                                  C.c_int32, C.POINTER(_P)]),
    "zsim_env_create_controlled": (C.c_int, [_P, C.c_size_t, C.POINTER(C.c_int64), C.c_int32, C.c_int32,
                                             C.POINTER(SimConfigC), c_double_p, C.c_int32, c_double_p, C.c_int32,
                                             C.c_int32, C.POINTER(_P)]),
    "zsim_env_get_rows": (C.c_int, [_P, c_int32_p, c_int32_p]),
    "zsim_controlled_expand": (C.c_int, [_P, C.c_size_t, C.POINTER(C.c_int64), C.c_int32, C.POINTER(SimConfigC),
                                         C.POINTER(_P), C.POINTER(C.c_size_t)]),
    "zsim_env_destroy": (C.c_int, [_P]),
    "zsim_stream_create": (C.c_int, [_P, C.c_size_t, C.c_int32, C.c_int32, C.POINTER(SimConfigC), c_double_p,
                                     C.c_int32, c_double_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                     C.POINTER(_P)]),
    "zsim_stream_num_batches": (C.c_int, [_P, C.POINTER(C.c_int64)]),
    "zsim_stream_next": (C.c_int, [_P, C.POINTER(_P)]),
    "zsim_stream_destroy": (C.c_int, [_P]),
    "zsim_episode_alloc": (C.c_int, [_P, C.c_int32, C.POINTER(EpisodeView)]),
    "zsim_episode_free": (C.c_int, [_P, C.POINTER(EpisodeView)]),
    "zsim_episode_bytes": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_size_t)]),
    "zsim_episode_carve": (C.c_int, [_P, C.c_int32, _P, C.POINTER(EpisodeView)]),
    "zsim_episode_copy": (C.c_int, [_P, C.POINTER(EpisodeView), C.POINTER(EpisodeView), C.c_int32, _P]),
    "zsim_rollout": (C.c_int, [_P, C.c_uint64, C.c_int32, c_int32_p, c_int32_p, C.c_int32, C.POINTER(EpisodeView),
                               C.POINTER(ObsView), C.POINTER(StateView), _P]),
    "zsim_score_defaults": (C.c_int, [C.POINTER(ScoreBounds), C.POINTER(ComfortWeights)]),
    "zsim_episode_metrics": (C.c_int, [_P, C.POINTER(EpisodeView), C.POINTER(ScoreBounds),
                                       C.POINTER(ComfortWeights), C.POINTER(MetricView), c_double_p, _P]),
    "zsim_aggregate_finalize": (C.c_int, [c_double_p, C.c_int32, c_double_p]),
    "zsim_env_get_info": (C.c_int, [_P, C.POINTER(EnvInfo)]),
    "zsim_env_get_scalars": (C.c_int, [_P, c_double_p, c_double_p, c_double_p]),
    "zsim_state_alloc": (C.c_int, [_P, C.POINTER(StateView)]),
    "zsim_state_free": (C.c_int, [_P, C.POINTER(StateView)]),
    "zsim_stepout_alloc": (C.c_int, [_P, C.POINTER(StepOutView)]),
    "zsim_stepout_free": (C.c_int, [_P, C.POINTER(StepOutView)]),
    "zsim_obs_alloc": (C.c_int, [_P, C.POINTER(ObsView)]),
    "zsim_obs_free": (C.c_int, [_P, C.POINTER(ObsView)]),
    "zsim_layout_bytes": (C.c_int, [_P, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "zsim_state_carve": (C.c_int, [_P, _P, C.POINTER(StateView)]),
    "zsim_stepout_carve": (C.c_int, [_P, _P, C.POINTER(StepOutView)]),
    "zsim_obs_carve": (C.c_int, [_P, _P, C.POINTER(ObsView)]),
    "zsim_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(_P)]),
    "zsim_host_free": (C.c_int, [_P]),
    "zsim_state_copy": (C.c_int, [_P, C.POINTER(StateView), C.POINTER(StateView), C.c_int32, _P]),
    "zsim_stepout_copy": (C.c_int, [_P, C.POINTER(StepOutView), C.POINTER(StepOutView), C.c_int32, _P]),
    "zsim_obs_copy": (C.c_int, [_P, C.POINTER(ObsView), C.POINTER(ObsView), C.c_int32, _P]),
    "zsim_reset": (C.c_int, [_P, C.c_uint64, C.POINTER(StateView), _P]),
    "zsim_step": (C.c_int, [_P, C.POINTER(StateView), c_int32_p, c_int32_p, C.POINTER(StateView),
                            C.POINTER(StepOutView), _P]),
    "zsim_observe": (C.c_int, [_P, C.POINTER(StateView), C.POINTER(ObsView), _P]),
    "zsim_step_observe": (C.c_int, [_P, C.POINTER(StateView), c_int32_p, c_int32_p, C.POINTER(StateView),
                                    C.POINTER(StepOutView), C.POINTER(ObsView), _P]),
    "zsim_episode_stats": (C.c_int, [_P, C.POINTER(StateView), C.POINTER(C.c_int64), _P]),
    "zsim_set_debug_topk": (C.c_int, [_P, c_int32_p]),
    "zsim_check_errors": (C.c_int, [_P, _P]),
    "zsim_set_launch_policy": (C.c_int, [_P, C.c_int32]),
    "zsim_reset_host": (C.c_int, [_P, C.c_uint64, C.POINTER(StateView)]),
    "zsim_step_host": (C.c_int, [_P, C.POINTER(StateView), c_int32_p, c_int32_p, C.POINTER(StateView),
                                 C.POINTER(StepOutView)]),
    "zsim_observe_host": (C.c_int, [_P, C.POINTER(StateView), C.POINTER(ObsView)]),
    "zsim_step_observe_host": (C.c_int, [_P, C.POINTER(StateView), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                         C.POINTER(StateView), C.POINTER(StepOutView), C.POINTER(ObsView)]),
    "zsim_stress_config_defaults": (C.c_int, [C.POINTER(StressConfigC)]),
    "zsim_stress_generate": (C.c_int, [C.POINTER(StressConfigC), C.c_uint64, C.POINTER(_P),
                                       C.POINTER(C.c_size_t)]),
    "zsim_free_buffer": (None, [_P]),
    "zsim_comm_available": (C.c_int, []),
    "zsim_comm_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "zsim_comm_init_rank": (C.c_int, [C.POINTER(C.c_uint8), C.c_int32, C.c_int32, C.c_int32, C.POINTER(_P)]),
    "zsim_comm_init_all": (C.c_int, [C.c_int32, c_int32_p, C.POINTER(_P)]),
    "zsim_comm_destroy": (C.c_int, [_P]),
    "zsim_comm_check": (C.c_int, [_P]),
    "zsim_stats_allreduce": (C.c_int, [_P, C.POINTER(C.c_int64), C.c_int32, _P]),
    "zsim_metric_sums_allgather": (C.c_int, [_P, c_double_p, C.c_int32, c_double_p, _P]),
    "zsim_comm_group": (C.c_int, [C.c_int32]),
    "zsim_env_create_stress": (C.c_int, [C.POINTER(StressConfigC), C.c_uint64, C.c_int32, C.POINTER(SimConfigC),
                                         C.c_int32, C.c_int32, C.POINTER(_P)]),
    "zsim_model_config_defaults": (C.c_int, [C.POINTER(ModelConfigC)]),
    "zsim_policy_param_count": (C.c_int, [C.POINTER(ModelConfigC), C.POINTER(C.c_int64)]),
    "zsim_policy_init_params": (C.c_int, [C.POINTER(ModelConfigC), C.c_uint64, c_float_p, C.c_int64]),
    "zsim_policy_create": (C.c_int, [C.POINTER(ModelConfigC), c_float_p, C.c_int64, C.c_int32, C.POINTER(_P)]),
    "zsim_policy_destroy": (C.c_int, [_P]),
    "zsim_policy_set_precision": (C.c_int, [_P, C.c_int32]),
    "zsim_policy_act_host": (C.c_int, [_P, C.POINTER(ObsView), C.c_int32, _P, C.c_int32, _P, _P, _P, _P]),
    "zsim_sequences_alloc": (C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(SequencesView)]),
    "zsim_sequences_free": (C.c_int, [_P, C.POINTER(SequencesView)]),
    "zsim_cut_sequences": (C.c_int, [_P, C.POINTER(EpisodeView), C.POINTER(ObsView), C.c_int32,
                                     C.POINTER(SequencesView), _P]),
    "zsim_rollout_policy": (C.c_int, [_P, _P, C.c_int32, C.c_uint64, C.c_int32, C.POINTER(EpisodeView),
                                      C.POINTER(ObsView), C.POINTER(StateView), _P]),
    "zsim_policy_act": (C.c_int, [_P, C.POINTER(ObsView), C.c_int32, _P, C.c_int32, _P, _P, _P, _P, _P, _P]),
}


class ZsimError(RuntimeError):
    """zsim::Error with its ErrorKind (common.hpp:13-22)."""

    KINDS = {1: "invalid_argument", 2: "config", 3: "io", 4: "runtime", 5: "cuda"}

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code
        self.kind = self.KINDS.get(code, "runtime")


def load_library(path: Path | str = LIB_PATH) -> C.CDLL:
    path = Path(path)
    if not path.exists():
        raise ImportError(
            f"native library {path} is missing; build it with `python paper_2312_15122_b200/build.py` "
            "(there is no CPU fallback on the product path)")
    lib = C.CDLL(str(path))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = load_library()


def check(code: int) -> None:
    if code != 0:
        raise ZsimError(code, lib.zsim_last_error().decode(errors="replace"))

"""Host-side mirror of the reference's ``zsim::sim::Env`` over the C-ABI.

Same method names, argument meaning and error behaviour as
``/root/reference/proj/src/core/simcore.hpp:191-245``:

* ``Env(batch, config, table)``      -> ``Env(zsim, indices, horizon, config, accel_bins, steer_bins)``
* ``init_state(seed)``                -> ``SimStateBatch``            (simcore.cpp:237-276)
* ``step(state, accel, steer, next, out)``                           (simcore.cpp:406-421)
* ``observe(state, obs)``                                             (simcore.cpp:540-552)
* accessors ``batch_size / horizon / dt / config / goal_s / initial_s / logged_progress``

plus a device fast path (``DeviceState`` / ``DeviceStepOut`` / ``DeviceObs``
and ``reset_device / step_device / observe_device / step_observe_device``)
whose buffers stay resident in HBM and whose launches are stream-ordered.
Errors raise ``ZsimError`` with the reference's ErrorKind.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, fields
from pathlib import Path

import numpy as np

from ._abi import (ComfortWeights, EnvInfo, EpisodeView, MetricView, ObsView, ScoreBounds, SequencesView, SimConfigC,
                   StateView,
                   StepOutView, StressConfigC, ZsimError, check, lib)

DONE_REASONS = ("none", "collision", "off_route", "red_light", "stop_line", "goal_reached")
ACTIVE_FEAT, AGENT_FEAT, ROAD_FEAT, ROUTE_FEAT, VALUE_FEAT = 9, 6, 12, 5, 2  # ObsSpec (simcore.hpp:60-72)


def event_bit(reason: int) -> int:
    """simcore.hpp:58."""
    return 1 << (reason - 1)


@dataclass
class SimConfig:
    """SimConfig (simcore.hpp:14-45) with dyn::Limits (dynamics.hpp:18-21) flattened."""
    wheelbase: float = 3.0
    ego_length: float = 4.7
    ego_width: float = 1.9
    ego_center_offset: float = 1.5
    delta_max: float = 0.55
    v_min: float = 0.0
    goal_radius: float = 2.0
    footprint_margin: float = 0.1
    stop_cross_speed: float = 0.5
    stop_zone: float = 2.0
    stop_slow_speed: float = 0.1
    disable_dones: bool = False
    w_progress: float = 1.0
    w_speed: float = 0.1
    w_lat: float = 0.02
    w_lon: float = 0.02
    terminal_penalty: float = 10.0
    n_agents: int = 16
    n_road: int = 128
    n_route: int = 64
    feature_radius: float = 100.0
    threads: int = 1

    def to_c(self) -> SimConfigC:
        c = SimConfigC()
        check(lib.zsim_sim_config_defaults(C.byref(c)))
        for f in fields(self):
            setattr(c, f.name, int(getattr(self, f.name)) if f.name in (
                "disable_dones", "n_agents", "n_road", "n_route", "threads") else float(getattr(self, f.name)))
        return c


def _take_bytes(addr: int, n: int) -> bytes:
    """Copy n bytes at addr (ctypes.string_at takes a C int size: > 2 GiB images need this)."""
    return np.ctypeslib.as_array((C.c_uint8 * n).from_address(addr)).tobytes() if n else b""


def _ptr(a: np.ndarray, ctype):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.POINTER(ctype))


def _addr(p) -> int:
    return C.cast(p, C.c_void_p).value or 0


def _np_at(addr: int, dtype, n: int) -> np.ndarray:
    dt = np.dtype(dtype)
    buf = (C.c_char * max(1, n * dt.itemsize)).from_address(addr)
    return np.frombuffer(buf, dtype=dt, count=n)


_STATE_FIELDS = (("x", np.float64, C.c_double), ("y", np.float64, C.c_double),
                 ("heading", np.float64, C.c_double), ("v", np.float64, C.c_double),
                 ("steering", np.float64, C.c_double), ("t", np.int32, C.c_int32), ("done", np.uint8, C.c_uint8),
                 ("reason", np.uint8, C.c_uint8), ("rng", np.uint64, C.c_uint64),
                 ("proj_s", np.float64, C.c_double), ("proj_d", np.float64, C.c_double),
                 ("proj_in_corridor", np.uint8, C.c_uint8), ("events", np.uint8, C.c_uint8),
                 ("stopped_flags", np.uint8, C.c_uint8))
_STEPOUT_FIELDS = (("reward", np.float32, C.c_float), ("event", np.uint8, C.c_uint8), ("s", np.float32, C.c_float),
                   ("a_lat", np.float32, C.c_float), ("a_lon", np.float32, C.c_float), ("v", np.float32, C.c_float))
_OBS_FIELDS = ("active", "agents", "road", "route", "value_only")


def _state_view(st) -> StateView:
    """View of any SoA state container (ours or an oracle's), by field name."""
    if isinstance(st, SimStateBatch):
        return st.view()
    v = StateView()
    for name, _, ct in _STATE_FIELDS:
        setattr(v, name, _ptr(getattr(st, name), ct))
    return v


def _stepout_view(so) -> StepOutView:
    if isinstance(so, StepOut):
        return so.view()
    v = StepOutView()
    for name, _, ct in _STEPOUT_FIELDS:
        setattr(v, name, _ptr(getattr(so, name), ct))
    return v


def _obs_view(ob) -> ObsView:
    if isinstance(ob, ObservationBatch):
        return ob.view()
    v = ObsView()
    for name in _OBS_FIELDS:
        setattr(v, name, _ptr(getattr(ob, name), C.c_float))
    return v


class _Pinned:
    """Page-locked host block from zsim_host_alloc, freed on collection."""

    def __init__(self, nbytes: int):
        p = C.c_void_p()
        check(lib.zsim_host_alloc(C.c_size_t(nbytes), C.byref(p)))
        self.addr = p.value
        self.nbytes = nbytes

    def __del__(self):
        if getattr(self, "addr", None):
            lib.zsim_host_free(C.c_void_p(self.addr))
            self.addr = None


class _CachedView:
    """The ctypes view of a batch container is built once and reused (the
    host-vector calls are per step; building 14 pointers each call cost ~0.1
    ms of Python per step).  Rebinding a field array drops the cached view;
    in-place writes (``st.x[...] = ...``) keep it valid."""

    _VIEW_FIELDS: tuple = ()

    def __setattr__(self, name, value):
        if name in self._VIEW_FIELDS:
            self.__dict__.pop("_view", None)
        object.__setattr__(self, name, value)

    def view(self):
        v = self.__dict__.get("_view")
        if v is None:
            v = self._build_view()
            self.__dict__["_view"] = v
        return v


class SimStateBatch(_CachedView):
    """SimStateBatch (simcore.hpp:107-121) as SoA numpy arrays."""

    _VIEW_FIELDS = tuple(f[0] for f in _STATE_FIELDS)

    def __init__(self, batch: int, total_stop_lines: int, arrays: dict | None = None, owner=None):
        self.batch = batch
        self.total_stop_lines = total_stop_lines
        self._owner = owner
        for name, dt, _ in _STATE_FIELDS:
            n = total_stop_lines if name == "stopped_flags" else batch
            a = arrays[name] if arrays is not None else np.zeros(max(n, 1), dtype=dt)
            setattr(self, name, a)

    @classmethod
    def pinned(cls, env: "Env") -> "SimStateBatch":
        blk = _Pinned(env.layout[0])
        v = StateView()
        check(lib.zsim_state_carve(env.handle, C.c_void_p(blk.addr), C.byref(v)))
        arrays = {}
        for name, dt, _ in _STATE_FIELDS:
            n = env.total_stop_lines if name == "stopped_flags" else env.batch_size()
            arrays[name] = _np_at(_addr(getattr(v, name)), dt, max(n, 1))
        return cls(env.batch_size(), env.total_stop_lines, arrays, owner=blk)

    def _build_view(self) -> StateView:
        v = StateView()
        for name, _, ct in _STATE_FIELDS:
            setattr(v, name, _ptr(getattr(self, name), ct))
        return v

    def copy(self) -> "SimStateBatch":
        s = SimStateBatch(self.batch, self.total_stop_lines)
        for name, _, _ in _STATE_FIELDS:
            getattr(s, name)[...] = getattr(self, name)
        return s

    def copy_from(self, other: "SimStateBatch") -> None:
        for name, _, _ in _STATE_FIELDS:
            getattr(self, name)[...] = getattr(other, name)


class StepOut(_CachedView):
    """StepOut (simcore.hpp:123-131)."""

    _VIEW_FIELDS = tuple(f[0] for f in _STEPOUT_FIELDS)

    def __init__(self, batch: int, arrays: dict | None = None, owner=None):
        self.batch = batch
        self._owner = owner
        for name, dt, _ in _STEPOUT_FIELDS:
            setattr(self, name, arrays[name] if arrays is not None else np.zeros(batch, dtype=dt))

    @classmethod
    def pinned(cls, env: "Env") -> "StepOut":
        blk = _Pinned(env.layout[1])
        v = StepOutView()
        check(lib.zsim_stepout_carve(env.handle, C.c_void_p(blk.addr), C.byref(v)))
        arrays = {name: _np_at(_addr(getattr(v, name)), dt, env.batch_size()) for name, dt, _ in _STEPOUT_FIELDS}
        return cls(env.batch_size(), arrays, owner=blk)

    def _build_view(self) -> StepOutView:
        v = StepOutView()
        for name, _, ct in _STEPOUT_FIELDS:
            setattr(v, name, _ptr(getattr(self, name), ct))
        return v


class ObservationBatch(_CachedView):
    """ObservationBatch (simcore.hpp:76-103): [B][slot][feat] f32 per modality."""

    _VIEW_FIELDS = _OBS_FIELDS

    def __init__(self, batch: int, n_agents: int, n_road: int, n_route: int, arrays: dict | None = None,
                 owner=None):
        self.batch = batch
        self.n_agents, self.n_road, self.n_route = n_agents, n_road, n_route
        self._owner = owner
        shapes = self.shapes()
        for name in _OBS_FIELDS:
            a = arrays[name] if arrays is not None else np.zeros(int(np.prod(shapes[name])), dtype=np.float32)
            setattr(self, name, a.reshape(shapes[name]))

    def shapes(self) -> dict:
        B = self.batch
        return {"active": (B, ACTIVE_FEAT), "agents": (B, self.n_agents, AGENT_FEAT),
                "road": (B, self.n_road, ROAD_FEAT), "route": (B, self.n_route, ROUTE_FEAT),
                "value_only": (B, VALUE_FEAT)}

    @classmethod
    def pinned(cls, env: "Env") -> "ObservationBatch":
        blk = _Pinned(env.layout[2])
        v = ObsView()
        check(lib.zsim_obs_carve(env.handle, C.c_void_p(blk.addr), C.byref(v)))
        cfg = env.config()
        tmp = cls(env.batch_size(), cfg.n_agents, cfg.n_road, cfg.n_route)
        arrays = {name: _np_at(_addr(getattr(v, name)), np.float32, getattr(tmp, name).size) for name in _OBS_FIELDS}
        return cls(env.batch_size(), cfg.n_agents, cfg.n_road, cfg.n_route, arrays, owner=blk)

    def _build_view(self) -> ObsView:
        v = ObsView()
        for name in _OBS_FIELDS:
            setattr(v, name, _ptr(getattr(self, name), C.c_float))
        return v

    @property
    def nbytes(self) -> int:
        return sum(getattr(self, n).nbytes for n in _OBS_FIELDS)


class _DeviceBuf:
    def __init__(self, env: "Env", view, free_fn):
        self.env = env
        self.v = view
        self._free = free_fn

    def close(self):
        if self._free is not None and self.env.handle:
            self._free(self.env.handle, C.byref(self.v))
        self._free = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceState(_DeviceBuf):
    pass


class DeviceStepOut(_DeviceBuf):
    pass


class DeviceObs(_DeviceBuf):
    pass


class DeviceEpisode(_DeviceBuf):
    """A device EpisodeBatch (zsim_episode_alloc)."""


EPISODE_BT = ("accel_idx", "steer_idx", "logp", "value", "reward", "s", "a_lat", "a_lon", "v", "done", "mask")
EPISODE_B = ("bootstrap", "terminal", "events", "initial_s", "logged_progress")
AGGREGATE_FIELDS = ("scenarios", "degenerate", "mean_score", "mean_relative_progress", "mean_progress_ratio_raw",
                    "mean_collision_free", "mean_off_route_free", "mean_stop_line_free",
                    "mean_traffic_light_free", "mean_comfort", "failure_rate", "goal_rate")


def aggregate_finalize(partials) -> dict:
    """metrics::aggregate from per-GPU partial sums ([n][12], summed in order)."""
    p = np.ascontiguousarray(np.atleast_2d(np.asarray(partials, dtype=np.float64)))
    out = np.zeros(12)
    check(lib.zsim_aggregate_finalize(_ptr(p, C.c_double), int(p.shape[0]), _ptr(out, C.c_double)))
    return dict(zip(AGGREGATE_FIELDS, out.tolist()))


def _stream(s) -> C.c_void_p:
    if s is None:
        return C.c_void_p(0)
    if hasattr(s, "cuda_stream"):
        return C.c_void_p(s.cuda_stream)
    return C.c_void_p(int(s))


class Env:
    """The batched log-replay environment on one B200 (simcore.hpp:188-245)."""

    def __init__(self, zsim, indices=None, horizon: int = 0, config: SimConfig | None = None,
                 accel_bins=None, steer_bins=None, device: int = 0, controlled: bool = False):
        """`controlled=True`: one row per controllable actor of every scenario
        ("all agents controlled"; see
        zsim_env_create_controlled in include/zsim_gpu.h and `rows`)."""
        if isinstance(zsim, (str, os.PathLike)):
            zsim = Path(zsim).read_bytes()
        self._bytes = bytes(zsim)
        self._config = config or SimConfig()
        cfg = self._config.to_c()
        idx = None
        n_idx = 0
        if indices is not None:
            arr = np.ascontiguousarray(np.asarray(indices, dtype=np.int64))
            idx, n_idx = arr.ctypes.data_as(C.POINTER(C.c_int64)), int(arr.size)
            self._idx_keep = arr
        ab = np.ascontiguousarray(accel_bins, dtype=np.float64) if accel_bins is not None else None
        sb = np.ascontiguousarray(steer_bins, dtype=np.float64) if steer_bins is not None else None
        h = C.c_void_p()
        buf = C.create_string_buffer(self._bytes, len(self._bytes))
        create = lib.zsim_env_create_controlled if controlled else lib.zsim_env_create
        check(create(C.cast(buf, C.c_void_p), C.c_size_t(len(self._bytes)), idx, n_idx, int(horizon),
                     C.byref(cfg), None if ab is None else _ptr(ab, C.c_double),
                     0 if ab is None else int(ab.size), None if sb is None else _ptr(sb, C.c_double),
                     0 if sb is None else int(sb.size), int(device), C.byref(h)))
        self.handle = h.value
        self._owned = True
        self._attach()

    @classmethod
    def from_stress(cls, stress: "StressConfig", seed: int = 7, horizon: int = 0, config: SimConfig | None = None,
                    device: int = 0, controlled: bool = False) -> "Env":
        """Env over stress scenarios generated on the host cores and staged
        directly (zsim_env_create_stress): same rows as
        ``Env(stress_scenarios(stress, seed), ...)`` without the ZSIM image."""
        self = cls.__new__(cls)
        self._bytes = b""
        self._config = config or SimConfig()
        cfg = self._config.to_c()
        sc = StressConfigC(**{f.name: getattr(stress, f.name) for f in fields(stress)})
        h = C.c_void_p()
        check(lib.zsim_env_create_stress(C.byref(sc), C.c_uint64(seed), int(horizon), C.byref(cfg), int(device),
                                         int(bool(controlled)), C.byref(h)))
        self.handle = h.value
        self._owned = True
        self._attach()
        return self

    @classmethod
    def _borrowed(cls, handle: int, config: SimConfig) -> "Env":
        """An Env over a handle owned elsewhere (a BatchStream batch)."""
        self = cls.__new__(cls)
        self._bytes = b""
        self._config = config
        self.handle = handle
        self._owned = False
        self._attach()
        return self

    def _attach(self) -> None:
        info = EnvInfo()
        check(lib.zsim_env_get_info(self.handle, C.byref(info)))
        self.info = info
        self.total_stop_lines = info.total_stop_lines
        B = info.batch
        self._goal_s = np.zeros(B)
        self._initial_s = np.zeros(B)
        self._logged = np.zeros(B)
        check(lib.zsim_env_get_scalars(self.handle, _ptr(self._goal_s, C.c_double), _ptr(self._initial_s, C.c_double),
                                       _ptr(self._logged, C.c_double)))
        sb_, so_, ob_ = C.c_size_t(), C.c_size_t(), C.c_size_t()
        check(lib.zsim_layout_bytes(self.handle, C.byref(sb_), C.byref(so_), C.byref(ob_)))
        self.layout = (sb_.value, so_.value, ob_.value)
        self.row_scenario = np.zeros(B, dtype=np.int32)
        self.row_actor = np.zeros(B, dtype=np.int32)
        check(lib.zsim_env_get_rows(self.handle, _ptr(self.row_scenario, C.c_int32), _ptr(self.row_actor, C.c_int32)))

    def close(self):
        if getattr(self, "handle", None):
            if getattr(self, "_owned", True):
                lib.zsim_env_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --- accessors (simcore.hpp:200-209) ---
    def batch_size(self) -> int:
        return self.info.batch

    def horizon(self) -> int:
        return self.info.horizon

    def dt(self) -> float:
        return self.info.dt

    def config(self) -> SimConfig:
        return self._config

    def goal_s(self, b: int) -> float:
        return float(self._goal_s[b])

    def initial_s(self, b: int) -> float:
        return float(self._initial_s[b])

    def logged_progress(self, b: int) -> float:
        return float(self._logged[b])

    @property
    def zero_accel_idx(self) -> int:
        return self.info.zero_accel_idx

    @property
    def zero_steer_idx(self) -> int:
        return self.info.zero_steer_idx

    # --- host-vector path (the drop-in overloads) ---
    def new_state(self, pinned: bool = False) -> SimStateBatch:
        return SimStateBatch.pinned(self) if pinned else SimStateBatch(self.batch_size(), self.total_stop_lines)

    def new_stepout(self, pinned: bool = False) -> StepOut:
        return StepOut.pinned(self) if pinned else StepOut(self.batch_size())

    def new_obs(self, pinned: bool = False) -> ObservationBatch:
        c = self._config
        return ObservationBatch.pinned(self) if pinned else ObservationBatch(self.batch_size(), c.n_agents, c.n_road,
                                                                             c.n_route)

    def init_state(self, seed: int, out: SimStateBatch | None = None) -> SimStateBatch:
        st = out or self.new_state()
        v = st.view()
        check(lib.zsim_reset_host(self.handle, C.c_uint64(seed), C.byref(v)))
        return st

    def step(self, state: SimStateBatch, accel_idx, steer_idx, next: SimStateBatch | None = None,
             out: StepOut | None = None):
        B = self.batch_size()
        a = np.ascontiguousarray(accel_idx, dtype=np.int32)
        s = np.ascontiguousarray(steer_idx, dtype=np.int32)
        if a.size != B or s.size != B or state.batch != B:
            raise ZsimError(1, "env_step: action/state shape mismatch")
        nxt = next if next is not None else self.new_state()
        so = out if out is not None else self.new_stepout()
        vin, vout, vso = _state_view(state), _state_view(nxt), _stepout_view(so)
        check(lib.zsim_step_host(self.handle, C.byref(vin), _ptr(a, C.c_int32), _ptr(s, C.c_int32), C.byref(vout),
                                 C.byref(vso)))
        return nxt, so

    def observe(self, state: SimStateBatch, obs: ObservationBatch | None = None) -> ObservationBatch:
        ob = obs if obs is not None else self.new_obs()
        vin, vo = _state_view(state), _obs_view(ob)
        check(lib.zsim_observe_host(self.handle, C.byref(vin), C.byref(vo)))
        return ob

    def step_observe(self, state: SimStateBatch, accel_idx, steer_idx, next: SimStateBatch | None = None,
                     out: StepOut | None = None, obs: ObservationBatch | None = None):
        """step followed by observe of the next state (the rollout loop body,
        simcore.cpp:590-609) in one host-vector call (zsim_step_observe_host):
        the same results as step() then observe(), one state upload, the
        observation streamed back while the kernel runs."""
        B = self.batch_size()
        a = np.ascontiguousarray(accel_idx, dtype=np.int32)
        s = np.ascontiguousarray(steer_idx, dtype=np.int32)
        if a.size != B or s.size != B or state.batch != B:
            raise ZsimError(1, "env_step: action/state shape mismatch")
        nxt = next if next is not None else self.new_state()
        so = out if out is not None else self.new_stepout()
        ob = obs if obs is not None else self.new_obs()
        vin, vout, vso, vo = _state_view(state), _state_view(nxt), _stepout_view(so), _obs_view(ob)
        check(lib.zsim_step_observe_host(self.handle, C.byref(vin), _ptr(a, C.c_int32), _ptr(s, C.c_int32),
                                         C.byref(vout), C.byref(vso), C.byref(vo)))
        return nxt, so, ob

    # --- device fast path ---
    def device_state(self) -> DeviceState:
        v = StateView()
        check(lib.zsim_state_alloc(self.handle, C.byref(v)))
        return DeviceState(self, v, lib.zsim_state_free)

    def device_stepout(self) -> DeviceStepOut:
        v = StepOutView()
        check(lib.zsim_stepout_alloc(self.handle, C.byref(v)))
        return DeviceStepOut(self, v, lib.zsim_stepout_free)

    def device_obs(self) -> DeviceObs:
        v = ObsView()
        check(lib.zsim_obs_alloc(self.handle, C.byref(v)))
        return DeviceObs(self, v, lib.zsim_obs_free)

    def reset_device(self, seed: int, out: DeviceState, stream=None) -> None:
        check(lib.zsim_reset(self.handle, C.c_uint64(seed), C.byref(out.v), _stream(stream)))

    def step_device(self, state: DeviceState, accel_ptr: int, steer_ptr: int, next: DeviceState,
                    out: DeviceStepOut, stream=None) -> None:
        check(lib.zsim_step(self.handle, C.byref(state.v), C.cast(C.c_void_p(accel_ptr), C.POINTER(C.c_int32)),
                            C.cast(C.c_void_p(steer_ptr), C.POINTER(C.c_int32)), C.byref(next.v), C.byref(out.v),
                            _stream(stream)))

    def observe_device(self, state: DeviceState, obs: DeviceObs, stream=None) -> None:
        check(lib.zsim_observe(self.handle, C.byref(state.v), C.byref(obs.v), _stream(stream)))

    def step_observe_device(self, state: DeviceState, accel_ptr: int, steer_ptr: int, next: DeviceState,
                            out: DeviceStepOut, obs: DeviceObs, stream=None) -> None:
        check(lib.zsim_step_observe(self.handle, C.byref(state.v),
                                    C.cast(C.c_void_p(accel_ptr), C.POINTER(C.c_int32)),
                                    C.cast(C.c_void_p(steer_ptr), C.POINTER(C.c_int32)), C.byref(next.v),
                                    C.byref(out.v), C.byref(obs.v), _stream(stream)))

    def episode_stats(self, state: DeviceState, out_ptr: int, stream=None) -> None:
        """int64[8] episode-stats vector of `state` into device memory `out_ptr`."""
        check(lib.zsim_episode_stats(self.handle, C.byref(state.v), C.cast(C.c_void_p(out_ptr),
                                                                           C.POINTER(C.c_int64)), _stream(stream)))

    # ---- device rollout recording + metrics ----
    def device_episode(self, horizon: int) -> DeviceEpisode:
        v = EpisodeView()
        check(lib.zsim_episode_alloc(self.handle, int(horizon), C.byref(v)))
        return DeviceEpisode(self, v, lib.zsim_episode_free)

    def rollout_device(self, seed: int, horizon: int, accel_ptr: int, steer_ptr: int, script_len: int,
                       episode: DeviceEpisode | None = None, obs: list | None = None,
                       final_state: DeviceState | None = None, stream=None) -> None:
        """Env::rollout(ScriptedPolicy) on the device: the script is a device
        int32 [script_len][B] pair read at each row's t.  `obs`: None or a list
        of horizon+1 DeviceObs (obs[0..T-1] and the final observation)."""
        ov = None
        if obs is not None:
            assert len(obs) == horizon + 1
            arr = (ObsView * (horizon + 1))(*[o.v for o in obs])
            ov = arr
        check(lib.zsim_rollout(self.handle, C.c_uint64(seed), int(horizon),
                               C.cast(C.c_void_p(accel_ptr), C.POINTER(C.c_int32)),
                               C.cast(C.c_void_p(steer_ptr), C.POINTER(C.c_int32)), int(script_len),
                               C.byref(episode.v) if episode is not None else None, ov,
                               C.byref(final_state.v) if final_state is not None else None, _stream(stream)))

    def rollout_policy_device(self, policy, seed: int, horizon: int, episode: DeviceEpisode | None = None,
                              obs: list | None = None, final_state: DeviceState | None = None, stream=None) -> None:
        """Env::rollout(NNPolicy) on the device (zsim_rollout_policy): the
        policy (paper_2312_15122_b200.NNPolicy) acts on every observation with
        the rows' rng streams; `obs` / `final_state` as rollout_device."""
        ov = None
        if obs is not None:
            assert len(obs) == horizon + 1
            ov = (ObsView * (horizon + 1))(*[o.v for o in obs])
        check(lib.zsim_rollout_policy(self.handle, policy.handle, int(policy.argmax), C.c_uint64(seed), int(horizon),
                                      C.byref(episode.v) if episode is not None else None, ov,
                                      C.byref(final_state.v) if final_state is not None else None, _stream(stream)))

    def cut_sequences_device(self, ep: DeviceEpisode, obs: list, seq_len: int, stream=None) -> dict:
        """train::cut_sequences (replay.cpp:8-52) of a recorded device episode
        (zsim_cut_sequences); `obs` the episode's observation list as
        rollout_device records it (obs[t] precedes step t).  Returns torch
        CUDA tensors sized for the maximum sequence count ("count" holds the
        number written): per-step [cap][L], obs_<modality> [cap][L][slot][feat],
        bootstrap / row / t0 [cap]."""
        import torch
        T, B, L = ep.v.horizon, self.info.batch, int(seq_len)
        assert len(obs) >= T
        cap = B * ((T + L - 1) // L) if L > 0 else 0
        cfg = self.config()
        dev = torch.device("cuda", self.info.device)
        t = {"accel_idx": torch.zeros(cap, L, dtype=torch.int32, device=dev),
             "steer_idx": torch.zeros(cap, L, dtype=torch.int32, device=dev),
             "logmu": torch.zeros(cap, L, device=dev), "reward": torch.zeros(cap, L, device=dev),
             "done": torch.zeros(cap, L, dtype=torch.uint8, device=dev),
             "mask": torch.zeros(cap, L, dtype=torch.uint8, device=dev),
             "bootstrap": torch.zeros(cap, device=dev), "row": torch.zeros(cap, dtype=torch.int32, device=dev),
             "t0": torch.zeros(cap, dtype=torch.int32, device=dev), "count": torch.zeros(1, dtype=torch.int32, device=dev),
             "obs_active": torch.zeros(cap, L, 9, device=dev),
             "obs_agents": torch.zeros(cap, L, cfg.n_agents, 6, device=dev),
             "obs_road": torch.zeros(cap, L, cfg.n_road, 12, device=dev),
             "obs_route": torch.zeros(cap, L, cfg.n_route, 5, device=dev),
             "obs_value_only": torch.zeros(cap, L, 2, device=dev)}
        v = SequencesView()
        v.capacity, v.seq_len = cap, L
        for f in ("active", "agents", "road", "route", "value_only"):
            setattr(v.obs, f, C.cast(C.c_void_p(t["obs_" + f].data_ptr()), C.POINTER(C.c_float)))
        for f in ("accel_idx", "steer_idx", "logmu", "reward", "done", "mask", "bootstrap", "row", "t0", "count"):
            setattr(v, f, C.cast(C.c_void_p(t[f].data_ptr()), type(getattr(v, f))))
        views = (ObsView * T)(*[o.v for o in obs[:T]])
        check(lib.zsim_cut_sequences(self.handle, C.byref(ep.v), views, L, C.byref(v), _stream(stream)))
        return t

    def download_episode(self, ep: DeviceEpisode) -> dict:
        """Host copy of a device EpisodeBatch: [B][T] and [B] numpy arrays."""
        B, T = self.info.batch, ep.v.horizon
        n = C.c_size_t()
        check(lib.zsim_episode_bytes(self.handle, T, C.byref(n)))
        buf = np.zeros(n.value, dtype=np.uint8)
        hv = EpisodeView()
        check(lib.zsim_episode_carve(self.handle, T, C.c_void_p(buf.ctypes.data), C.byref(hv)))
        check(lib.zsim_episode_copy(self.handle, C.byref(hv), C.byref(ep.v), 1, None))
        check(lib.zsim_check_errors(self.handle, None))
        out = {}
        types = {"accel_idx": np.int32, "steer_idx": np.int32, "done": np.uint8, "mask": np.uint8,
                 "terminal": np.uint8, "events": np.uint8}
        for f in EPISODE_BT + EPISODE_B:
            dt = types.get(f, np.float32)
            cnt = B * T if f in EPISODE_BT else B
            addr = C.cast(getattr(hv, f), C.c_void_p).value
            out[f] = np.frombuffer((C.c_char * (cnt * np.dtype(dt).itemsize)).from_address(addr),
                                   dtype=dt).copy().reshape((B, T) if f in EPISODE_BT else (B,))
        return out

    def episode_metrics(self, ep: DeviceEpisode, rows: bool = True, bounds: dict | None = None,
                        weights: dict | None = None):
        """metrics::score_episode per row (host dict of [B] arrays, or None)
        and this GPU's Aggregate partial sums (12 doubles)."""
        import torch  # device buffers for the outputs
        B = self.info.batch
        dev = torch.device("cuda", self.info.device)
        sums = torch.zeros(12, dtype=torch.float64, device=dev)
        bb, cw = ScoreBounds(), ComfortWeights()
        check(lib.zsim_score_defaults(C.byref(bb), C.byref(cw)))
        for k, v in (bounds or {}).items():
            setattr(bb, k, v)
        for k, v in (weights or {}).items():
            setattr(cw, k, v)
        mv = MetricView()
        keep = {}
        if rows:
            for name, ct in MetricView._fields_:
                t = torch.zeros(B, dtype=torch.float64 if ct is not C.POINTER(C.c_uint8) else torch.uint8,
                                device=dev)
                keep[name] = t
                setattr(mv, name, C.cast(C.c_void_p(t.data_ptr()), ct))
        check(lib.zsim_episode_metrics(self.handle, C.byref(ep.v), C.byref(bb), C.byref(cw),
                                       C.byref(mv) if rows else None,
                                       C.cast(C.c_void_p(sums.data_ptr()), C.POINTER(C.c_double)), None))
        torch.cuda.synchronize(dev)
        per_row = {k: v.cpu().numpy() for k, v in keep.items()} if rows else None
        return per_row, sums.cpu().numpy()

    def set_debug_topk(self, dev_ptr: int | None) -> None:
        check(lib.zsim_set_debug_topk(self.handle, C.cast(C.c_void_p(dev_ptr or 0), C.POINTER(C.c_int32))))

    def set_launch_policy(self, policy: int) -> None:
        """0 automatic, 1 fused kernel, 2 split observation kernels (identical results)."""
        check(lib.zsim_set_launch_policy(self.handle, int(policy)))
        check(lib.zsim_env_get_info(self.handle, C.byref(self.info)))

    def check_errors(self, stream=None) -> None:
        check(lib.zsim_check_errors(self.handle, _stream(stream)))

    def download_state(self, dev: DeviceState, host: SimStateBatch | None = None, stream=None) -> SimStateBatch:
        st = host or self.new_state()
        v = st.view()
        check(lib.zsim_state_copy(self.handle, C.byref(v), C.byref(dev.v), 1, _stream(stream)))
        return st

    def upload_state(self, host: SimStateBatch, dev: DeviceState, stream=None) -> None:
        v = _state_view(host)
        check(lib.zsim_state_copy(self.handle, C.byref(dev.v), C.byref(v), 0, _stream(stream)))

    def download_stepout(self, dev: DeviceStepOut, host: StepOut | None = None, stream=None) -> StepOut:
        so = host or self.new_stepout()
        v = so.view()
        check(lib.zsim_stepout_copy(self.handle, C.byref(v), C.byref(dev.v), 1, _stream(stream)))
        return so

    def download_obs(self, dev: DeviceObs, host: ObservationBatch | None = None, stream=None) -> ObservationBatch:
        ob = host or self.new_obs()
        v = ob.view()
        check(lib.zsim_obs_copy(self.handle, C.byref(v), C.byref(dev.v), 1, _stream(stream)))
        return ob


@dataclass
class StressConfig:
    """Synthetic stress-scenario shape; see include/zsim_gpu.h."""
    count: int = 64
    num_steps: int = 92
    agents: int = 32
    road_points: int = 2048
    lanes: int = 4
    lane_vertices: int = 64
    dt: float = 0.1
    speed_limit: float = 10.0
    lane_width: float = 3.5
    first_index: int = 0
    flags: int = 0  # bit 0: C2 actors (all agents valid, same-direction route lanes)


STRESS_C2 = 1


def stress_scenarios(cfg: StressConfig, seed: int = 7) -> bytes:
    """ZSIM container image of `cfg.count` stress scenarios (host-only call)."""
    c = StressConfigC(**{f.name: getattr(cfg, f.name) for f in fields(cfg)})
    p = C.c_void_p()
    n = C.c_size_t()
    check(lib.zsim_stress_generate(C.byref(c), C.c_uint64(seed), C.byref(p), C.byref(n)))
    try:
        return _take_bytes(p.value, n.value)
    finally:
        lib.zsim_free_buffer(p)


class BatchStream:
    """scenario::BatchStream (scenario_stream.hpp:12-40) feeding device Envs:
    iterate to get one Env per batch; batch k+1 is decoded, staged and
    uploaded (pinned buffer, copy stream) while batch k is simulated.  Each
    Env is valid until the next batch is requested."""

    def __init__(self, zsim, batch_size: int, horizon: int = 0, config: SimConfig | None = None,
                 accel_bins=None, steer_bins=None, device: int = 0, prefetch: bool = True, controlled: bool = False):
        if isinstance(zsim, (str, os.PathLike)):
            zsim = Path(zsim).read_bytes()
        self._config = config or SimConfig()
        cfg = self._config.to_c()
        ab = np.ascontiguousarray(accel_bins, dtype=np.float64) if accel_bins is not None else None
        sb = np.ascontiguousarray(steer_bins, dtype=np.float64) if steer_bins is not None else None
        buf = C.create_string_buffer(bytes(zsim), len(zsim))
        h = C.c_void_p()
        check(lib.zsim_stream_create(C.cast(buf, C.c_void_p), C.c_size_t(len(zsim)), int(batch_size), int(horizon),
                                     C.byref(cfg), None if ab is None else _ptr(ab, C.c_double),
                                     0 if ab is None else int(ab.size), None if sb is None else _ptr(sb, C.c_double),
                                     0 if sb is None else int(sb.size), int(device), int(bool(prefetch)),
                                     int(bool(controlled)), C.byref(h)))
        self.handle = h.value
        self._env = None

    def __len__(self) -> int:
        n = C.c_int64()
        check(lib.zsim_stream_num_batches(self.handle, C.byref(n)))
        return n.value

    def __iter__(self):
        return self

    def __next__(self) -> "Env":
        if self._env is not None:
            self._env.handle = None  # the stream destroys it on the next call
        h = C.c_void_p()
        check(lib.zsim_stream_next(self.handle, C.byref(h)))
        if not h.value:
            self._env = None
            raise StopIteration
        self._env = Env._borrowed(h.value, self._config)
        return self._env

    def close(self):
        if getattr(self, "handle", None):
            if self._env is not None:
                self._env.handle = None
            lib.zsim_stream_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def controlled_expand(zsim: bytes, indices=None, config: SimConfig | None = None) -> bytes:
    """The per-row scenarios of a controlled Env (row order) as a ZSIM image:
    the reference Env over these is the oracle for Env(controlled=True)."""
    cfg = (config or SimConfig()).to_c()
    idx, n_idx = None, 0
    if indices is not None:
        arr = np.ascontiguousarray(np.asarray(indices, dtype=np.int64))
        idx, n_idx = arr.ctypes.data_as(C.POINTER(C.c_int64)), int(arr.size)
    buf = C.create_string_buffer(bytes(zsim), len(zsim))
    p = C.c_void_p()
    n = C.c_size_t()
    check(lib.zsim_controlled_expand(C.cast(buf, C.c_void_p), C.c_size_t(len(zsim)), idx, n_idx, C.byref(cfg),
                                     C.byref(p), C.byref(n)))
    try:
        return _take_bytes(p.value, n.value)
    finally:
        lib.zsim_free_buffer(p)


def random_actions(steps: int, batch: int, seed: int = 123, num_accel: int = 7, num_steer: int = 5):
    """Fixed [steps][batch] int32 action tensors, uniform over the bins from a
    splitmix64 stream (common.hpp:28-44), as the BASELINE plan prescribes."""
    n = steps * batch * 2
    g = 0x9E3779B97F4A7C15
    state = (seed + g) & 0xFFFFFFFFFFFFFFFF
    idx = np.arange(1, n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(state) + idx * np.uint64(g)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    z = z.reshape(steps, batch, 2)
    accel = (z[..., 0] % np.uint64(num_accel)).astype(np.int32)
    steer = (z[..., 1] % np.uint64(num_steer)).astype(np.int32)
    return np.ascontiguousarray(accel), np.ascontiguousarray(steer)

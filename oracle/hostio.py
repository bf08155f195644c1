"""TEST INFRASTRUCTURE: host-side containers and ctypes views for the oracles.

The oracles (``refpy`` over ``oracle/_ref/libzsim_ref.so``, ``portpy`` over
the C restatement) speak the plain-C structs of ``include/zsim_gpu.h``
(``zsim_sim_config``, ``zsim_state_view``, ``zsim_stepout_view``,
``zsim_obs_view``) -- header-only types, declared again here so that nothing
under ``oracle/`` imports the product package or maps ``libzsim_gpu.so``
(the reference arm of ``bench.py`` must run the reference alone).

The containers mirror the reference's SoA batches (``simcore.hpp:76-131``);
the product's ``Env`` accepts them (it reads the arrays by field name), so a
parity test can resynchronise the device from an oracle state.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

c_double_p = C.POINTER(C.c_double)
c_float_p = C.POINTER(C.c_float)
c_int32_p = C.POINTER(C.c_int32)
c_uint8_p = C.POINTER(C.c_uint8)
c_uint64_p = C.POINTER(C.c_uint64)

ACTIVE_FEAT, AGENT_FEAT, ROAD_FEAT, ROUTE_FEAT, VALUE_FEAT = 9, 6, 12, 5, 2  # ObsSpec (simcore.hpp:60-72)


class SimConfigC(C.Structure):
    """zsim_sim_config (include/zsim_gpu.h) = SimConfig (simcore.hpp:14-45)."""
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


# SimConfig defaults (simcore.hpp:14-45, dynamics.hpp:18-21)
_CONFIG_DEFAULTS = dict(wheelbase=3.0, ego_length=4.7, ego_width=1.9, ego_center_offset=1.5, delta_max=0.55,
                        v_min=0.0, goal_radius=2.0, footprint_margin=0.1, stop_cross_speed=0.5, stop_zone=2.0,
                        stop_slow_speed=0.1, disable_dones=False, w_progress=1.0, w_speed=0.1, w_lat=0.02,
                        w_lon=0.02, terminal_penalty=10.0, n_agents=16, n_road=128, n_route=64,
                        feature_radius=100.0, threads=1)
_INT_FIELDS = ("disable_dones", "n_agents", "n_road", "n_route", "threads")


class OracleConfig:
    """Plain SimConfig for the oracles; any object with SimConfig's attribute
    names (e.g. the product's ``SimConfig``) converts through ``config_c``."""

    def __init__(self, **kw):
        for k, v in _CONFIG_DEFAULTS.items():
            setattr(self, k, kw.pop(k, v))
        if kw:
            raise TypeError(f"unknown SimConfig fields {sorted(kw)}")


def config_c(cfg) -> SimConfigC:
    cfg = cfg if cfg is not None else OracleConfig()
    c = SimConfigC()
    for k, d in _CONFIG_DEFAULTS.items():
        v = getattr(cfg, k, d)
        setattr(c, k, int(v) if k in _INT_FIELDS else float(v))
    return c


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


STATE_FIELDS = (("x", np.float64, C.c_double), ("y", np.float64, C.c_double),
                ("heading", np.float64, C.c_double), ("v", np.float64, C.c_double),
                ("steering", np.float64, C.c_double), ("t", np.int32, C.c_int32), ("done", np.uint8, C.c_uint8),
                ("reason", np.uint8, C.c_uint8), ("rng", np.uint64, C.c_uint64),
                ("proj_s", np.float64, C.c_double), ("proj_d", np.float64, C.c_double),
                ("proj_in_corridor", np.uint8, C.c_uint8), ("events", np.uint8, C.c_uint8),
                ("stopped_flags", np.uint8, C.c_uint8))
STEPOUT_FIELDS = (("reward", np.float32, C.c_float), ("event", np.uint8, C.c_uint8), ("s", np.float32, C.c_float),
                  ("a_lat", np.float32, C.c_float), ("a_lon", np.float32, C.c_float), ("v", np.float32, C.c_float))
OBS_FIELDS = ("active", "agents", "road", "route", "value_only")


def ptr(a: np.ndarray, ctype):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.POINTER(ctype))


class State:
    """SimStateBatch (simcore.hpp:107-121), SoA numpy arrays."""

    def __init__(self, batch: int, total_stop_lines: int):
        self.batch, self.total_stop_lines = batch, total_stop_lines
        for name, dt, _ in STATE_FIELDS:
            n = total_stop_lines if name == "stopped_flags" else batch
            setattr(self, name, np.zeros(max(n, 1), dtype=dt))

    def view(self) -> StateView:
        v = StateView()
        for name, _, ct in STATE_FIELDS:
            setattr(v, name, ptr(getattr(self, name), ct))
        return v

    def copy(self) -> "State":
        s = State(self.batch, self.total_stop_lines)
        for name, _, _ in STATE_FIELDS:
            getattr(s, name)[...] = getattr(self, name)
        return s


class Out:
    """StepOut (simcore.hpp:123-131)."""

    def __init__(self, batch: int):
        self.batch = batch
        for name, dt, _ in STEPOUT_FIELDS:
            setattr(self, name, np.zeros(batch, dtype=dt))

    def view(self) -> StepOutView:
        v = StepOutView()
        for name, _, ct in STEPOUT_FIELDS:
            setattr(v, name, ptr(getattr(self, name), ct))
        return v


class Obs:
    """ObservationBatch (simcore.hpp:76-103): [B][slot][feat] f32."""

    def __init__(self, batch: int, n_agents: int, n_road: int, n_route: int):
        self.batch, self.n_agents, self.n_road, self.n_route = batch, n_agents, n_road, n_route
        self.active = np.zeros((batch, ACTIVE_FEAT), np.float32)
        self.agents = np.zeros((batch, n_agents, AGENT_FEAT), np.float32)
        self.road = np.zeros((batch, n_road, ROAD_FEAT), np.float32)
        self.route = np.zeros((batch, n_route, ROUTE_FEAT), np.float32)
        self.value_only = np.zeros((batch, VALUE_FEAT), np.float32)

    def view(self) -> ObsView:
        v = ObsView()
        for name in OBS_FIELDS:
            setattr(v, name, ptr(getattr(self, name), C.c_float))
        return v


def random_actions(steps: int, batch: int, seed: int = 123, num_accel: int = 7, num_steer: int = 5):
    """The benchmark's fixed [steps][batch] action tensors: splitmix64
    (common.hpp:28-44) draws, two per (step, row), reduced modulo the bin
    counts.  Same stream as the product's ``random_actions``."""
    n = steps * batch * 2
    g = 0x9E3779B97F4A7C15
    idx = np.arange(1, n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64((seed + g) & 0xFFFFFFFFFFFFFFFF) + idx * np.uint64(g)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    z = z.reshape(steps, batch, 2)
    return (np.ascontiguousarray((z[..., 0] % np.uint64(num_accel)).astype(np.int32)),
            np.ascontiguousarray((z[..., 1] % np.uint64(num_steer)).astype(np.int32)))


def state_view(st) -> StateView:
    """View of any SoA state container (an oracle's or the product's), by field name."""
    v = StateView()
    for name, _, ct in STATE_FIELDS:
        setattr(v, name, ptr(getattr(st, name), ct))
    return v

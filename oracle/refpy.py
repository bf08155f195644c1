"""TEST INFRASTRUCTURE: Python handle on the reference simulator compiled in
place (oracle/_ref/libzsim_ref.so, built by oracle/build_oracle.py from
/root/reference/proj/src/core without copying).  Mirrors the product's
host API so parity tests read the same on both sides.  Never imported by the
product path.
"""
from __future__ import annotations

import ctypes as C
import os
import tempfile
from pathlib import Path

import numpy as np

from oracle.hostio import Obs, ObsView, OracleConfig, Out, SimConfigC, State, StateView, StepOutView, config_c
from oracle.hostio import ptr as _ptr
from oracle.hostio import state_view

HERE = Path(__file__).resolve().parent
REF_LIB = HERE / "_ref" / "libzsim_ref.so"

_P = C.c_void_p
_SIGS = {
    "zref_last_error": (C.c_char_p, []),
    "zref_env_create": (C.c_int, [C.c_char_p, C.POINTER(C.c_int64), C.c_int32, C.c_int32, C.POINTER(SimConfigC),
                                  C.POINTER(_P)]),
    "zref_env_destroy": (None, [_P]),
    "zref_env_info": (C.c_int, [_P, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "zref_scalars": (C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "zref_init_state": (C.c_int, [_P, C.c_uint64, C.POINTER(StateView)]),
    "zref_step": (C.c_int, [_P, C.POINTER(StateView), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                            C.POINTER(StateView), C.POINTER(StepOutView)]),
    "zref_observe": (C.c_int, [_P, C.POINTER(StateView), C.POINTER(ObsView)]),
    "zref_validate": (C.c_int, [C.c_char_p, C.c_int64, C.c_char_p, C.c_int32]),
    "zref_generate": (C.c_int, [C.c_int32, C.c_int32, C.c_double, C.c_uint64, C.c_char_p]),
    "zref_recover_actions": (C.c_int, [C.c_char_p, C.c_int64, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                       C.c_int32, C.POINTER(C.c_int32)]),
    "zref_aggregate": (C.c_int, [C.c_int32, C.c_int32, C.c_double, C.POINTER(C.c_float), C.POINTER(C.c_float),
                                 C.POINTER(C.c_float), C.POINTER(C.c_uint8), C.POINTER(C.c_uint8),
                                 C.POINTER(C.c_float), C.POINTER(C.c_float), C.POINTER(C.c_double)]),
    "zref_rollout": (C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_uint64,
                               C.POINTER(C.c_int32), C.POINTER(C.c_int32)] + [C.POINTER(C.c_float)] * 7
                     + [C.POINTER(C.c_uint8)] * 2 + [C.POINTER(C.c_float), C.POINTER(C.c_uint8),
                                                     C.POINTER(C.c_uint8), C.POINTER(C.c_float),
                                                     C.POINTER(C.c_float)]),
    "zref_rollout_cut": (C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_uint64,
                                   C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                   C.POINTER(C.c_float), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                   C.POINTER(C.c_float), C.POINTER(C.c_float), C.POINTER(C.c_uint8),
                                   C.POINTER(C.c_uint8)] + [C.POINTER(C.c_float)] * 5),
    "zref_bench_step": (C.c_int, [C.c_char_p, C.POINTER(C.c_int32), C.c_int32, C.c_int32, C.c_int32,
                                  C.POINTER(SimConfigC), C.POINTER(C.c_double)]),
    "zref_bench": (C.c_int, [C.c_char_p, C.c_int32, C.c_int32, C.POINTER(SimConfigC), C.c_int32, C.c_int32,
                             C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_uint64,
                             C.POINTER(C.c_double)]),
}

_lib = None


def available() -> bool:
    return REF_LIB.exists()


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not REF_LIB.exists():
            raise FileNotFoundError(f"{REF_LIB} not built (needs /root/reference; run oracle/build_oracle.py)")
        _lib = C.CDLL(str(REF_LIB))
        for n, (r, a) in _SIGS.items():
            f = getattr(_lib, n)
            f.restype = r
            f.argtypes = a
    return _lib


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def _check(code: int) -> None:
    if code != 0:
        raise RefError(code, lib().zref_last_error().decode(errors="replace"))


def _as_path(zsim) -> tuple[str, object]:
    """Reference Dataset reads files; spill in-memory images to a temp file."""
    if isinstance(zsim, (str, os.PathLike)):
        return str(zsim), None
    tf = tempfile.NamedTemporaryFile(suffix=".zsim", delete=False)
    tf.write(bytes(zsim))
    tf.close()
    return tf.name, tf


class RefEnv:
    """The reference zsim::sim::Env (simcore.hpp:191-245) over the same inputs."""

    def __init__(self, zsim, indices=None, horizon: int = 0, config=None):
        self._path, self._tmp = _as_path(zsim)
        self._config = config or OracleConfig()
        cfg = config_c(self._config)
        idx, n = None, 0
        if indices is not None:
            self._idx = np.ascontiguousarray(np.asarray(indices, dtype=np.int64))
            idx, n = self._idx.ctypes.data_as(C.POINTER(C.c_int64)), int(self._idx.size)
        h = C.c_void_p()
        _check(lib().zref_env_create(self._path.encode(), idx, n, int(horizon), C.byref(cfg), C.byref(h)))
        self.handle = h.value
        b, hz, ts = C.c_int32(), C.c_int32(), C.c_int32()
        _check(lib().zref_env_info(self.handle, C.byref(b), C.byref(hz), C.byref(ts)))
        self.batch, self.horizon, self.total_stop_lines = b.value, hz.value, ts.value

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                lib().zref_env_destroy(self.handle)
                self.handle = None
            if getattr(self, "_tmp", None) is not None:
                os.unlink(self._path)
                self._tmp = None
        except Exception:
            pass

    def batch_size(self) -> int:
        return self.batch

    def scalars(self):
        g, i, l = np.zeros(self.batch), np.zeros(self.batch), np.zeros(self.batch)
        _check(lib().zref_scalars(self.handle, _ptr(g, C.c_double), _ptr(i, C.c_double), _ptr(l, C.c_double)))
        return g, i, l

    def new_state(self) -> State:
        return State(self.batch, self.total_stop_lines)

    def init_state(self, seed: int) -> State:
        st = self.new_state()
        v = state_view(st)
        _check(lib().zref_init_state(self.handle, C.c_uint64(seed), C.byref(v)))
        return st

    def step(self, state: State, accel, steer):
        a = np.ascontiguousarray(accel, dtype=np.int32)
        s = np.ascontiguousarray(steer, dtype=np.int32)
        nxt, so = self.new_state(), Out(self.batch)
        vi, vo, vs = state_view(state), nxt.view(), so.view()
        _check(lib().zref_step(self.handle, C.byref(vi), _ptr(a, C.c_int32), _ptr(s, C.c_int32), C.byref(vo),
                               C.byref(vs)))
        return nxt, so

    def observe(self, state: State) -> Obs:
        c = self._config
        ob = Obs(self.batch, c.n_agents, c.n_road, c.n_route)
        vi, vo = state_view(state), ob.view()
        _check(lib().zref_observe(self.handle, C.byref(vi), C.byref(vo)))
        return ob

    def rollout(self, horizon: int, accel, steer, seed: int = 42) -> dict:
        """Env::rollout with ScriptedPolicy over a per-row script ([B][L] indices):
        every EpisodeBatch array ([B][T] / [B])."""
        B = self.batch
        a = np.ascontiguousarray(accel, dtype=np.int32)
        s = np.ascontiguousarray(steer, dtype=np.int32)
        assert a.shape[0] == B and a.shape == s.shape
        L = a.shape[1]
        o = {k: np.zeros((B, horizon), dtype=dt) for k, dt in (
            ("accel_idx", np.int32), ("steer_idx", np.int32), ("logp", np.float32), ("value", np.float32),
            ("reward", np.float32), ("s", np.float32), ("a_lat", np.float32), ("a_lon", np.float32),
            ("v", np.float32), ("done", np.uint8), ("mask", np.uint8))}
        o.update({k: np.zeros(B, dtype=dt) for k, dt in (
            ("bootstrap", np.float32), ("terminal", np.uint8), ("events", np.uint8), ("initial_s", np.float32),
            ("logged_progress", np.float32))})
        P = lambda k, ct: _ptr(o[k], ct)  # noqa: E731
        _check(lib().zref_rollout(
            self.handle, int(horizon), int(L), _ptr(a, C.c_int32), _ptr(s, C.c_int32), C.c_uint64(seed),
            P("accel_idx", C.c_int32), P("steer_idx", C.c_int32), P("logp", C.c_float), P("value", C.c_float),
            P("reward", C.c_float), P("s", C.c_float), P("a_lat", C.c_float), P("a_lon", C.c_float),
            P("v", C.c_float), P("done", C.c_uint8), P("mask", C.c_uint8), P("bootstrap", C.c_float),
            P("terminal", C.c_uint8), P("events", C.c_uint8), P("initial_s", C.c_float),
            P("logged_progress", C.c_float)))
        return o


def _rollout_cut(self, horizon: int, accel, steer, seq_len: int, seed: int = 42) -> dict:
    """Env::rollout(ScriptedPolicy) then train::cut_sequences (replay.cpp:8-52)
    in the REFERENCE: the written sequences as numpy arrays."""
    B = self.batch
    a = np.ascontiguousarray(accel, dtype=np.int32)
    s = np.ascontiguousarray(steer, dtype=np.int32)
    L = a.shape[1]
    cap = B * ((horizon + seq_len - 1) // seq_len)
    cnt = np.zeros(1, np.int32)
    o = {"row": np.zeros(cap, np.int32), "bootstrap": np.zeros(cap, np.float32),
         "accel_idx": np.zeros((cap, seq_len), np.int32), "steer_idx": np.zeros((cap, seq_len), np.int32),
         "logmu": np.zeros((cap, seq_len), np.float32), "reward": np.zeros((cap, seq_len), np.float32),
         "done": np.zeros((cap, seq_len), np.uint8), "mask": np.zeros((cap, seq_len), np.uint8),
         "obs_active": np.zeros((cap, seq_len, 9), np.float32),
         "obs_agents": np.zeros((cap, seq_len, self._config.n_agents, 6), np.float32),
         "obs_road": np.zeros((cap, seq_len, self._config.n_road, 12), np.float32),
         "obs_route": np.zeros((cap, seq_len, self._config.n_route, 5), np.float32),
         "obs_value_only": np.zeros((cap, seq_len, 2), np.float32)}
    P = lambda k, ct: _ptr(o[k], ct)  # noqa: E731
    _check(lib().zref_rollout_cut(
        self.handle, int(horizon), int(L), _ptr(a, C.c_int32), _ptr(s, C.c_int32), C.c_uint64(seed), int(seq_len),
        int(cap), _ptr(cnt, C.c_int32), P("row", C.c_int32), P("bootstrap", C.c_float), P("accel_idx", C.c_int32),
        P("steer_idx", C.c_int32), P("logmu", C.c_float), P("reward", C.c_float), P("done", C.c_uint8),
        P("mask", C.c_uint8), P("obs_active", C.c_float), P("obs_agents", C.c_float), P("obs_road", C.c_float),
        P("obs_route", C.c_float), P("obs_value_only", C.c_float)))
    n = int(cnt[0])
    return {"count": n, **{k: v[:n] for k, v in o.items()}}


RefEnv.rollout_cut = _rollout_cut


def validate(zsim, index: int) -> str:
    path, tmp = _as_path(zsim)
    try:
        buf = C.create_string_buffer(1024)
        _check(lib().zref_validate(path.encode(), int(index), buf, 1024))
        return buf.value.decode()
    finally:
        if tmp is not None:
            os.unlink(path)


def generate(count: int, seed: int, num_steps: int = 92, density: float = 0.5) -> bytes:
    """Reference generate_synthetic + write_file -> ZSIM bytes."""
    with tempfile.TemporaryDirectory() as d:
        p = Path(d) / "gen.zsim"
        _check(lib().zref_generate(int(count), int(num_steps), float(density), C.c_uint64(seed), str(p).encode()))
        return p.read_bytes()


def recover_actions(zsim, index: int):
    path, tmp = _as_path(zsim)
    try:
        cap = 4096
        a = np.zeros(cap, np.int32)
        s = np.zeros(cap, np.int32)
        n = C.c_int32()
        _check(lib().zref_recover_actions(path.encode(), int(index), _ptr(a, C.c_int32), _ptr(s, C.c_int32), cap,
                                          C.byref(n)))
        return a[:n.value].copy(), s[:n.value].copy()
    finally:
        if tmp is not None:
            os.unlink(path)


def aggregate(s, a_lat, a_lon, mask, events, initial_s, logged_progress, dt: float) -> np.ndarray:
    """metrics::score_episode + aggregate over recorded [B][T] traces (12 doubles)."""
    B, T = s.shape
    out = np.zeros(12)
    arrs = [np.ascontiguousarray(x, dtype=np.float32) for x in (s, a_lat, a_lon)]
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    ev = np.ascontiguousarray(events, dtype=np.uint8)
    i0 = np.ascontiguousarray(initial_s, dtype=np.float32)
    lp = np.ascontiguousarray(logged_progress, dtype=np.float32)
    _check(lib().zref_aggregate(B, T, float(dt), *[_ptr(x, C.c_float) for x in arrs], _ptr(m, C.c_uint8),
                                _ptr(ev, C.c_uint8), _ptr(i0, C.c_float), _ptr(lp, C.c_float),
                                _ptr(out, C.c_double)))
    return out


def bench(zsim, n_rows: int, horizon: int, config, threads: int, warmup: int, steps: int, accel,
          steer, seed: int = 42) -> float:
    """Wall seconds of `steps` timed observe+step iterations over `n_rows` rows
    on `threads` shards; `accel`/`steer` are [episode_len][n_rows] and the
    state is re-initialised every episode_len steps."""
    path, tmp = _as_path(zsim)
    try:
        a = np.ascontiguousarray(accel, dtype=np.int32)
        s = np.ascontiguousarray(steer, dtype=np.int32)
        assert a.shape[1] == n_rows
        cfg = config_c(config)
        out = C.c_double()
        _check(lib().zref_bench(path.encode(), int(n_rows), int(horizon), C.byref(cfg), int(threads), int(warmup),
                                int(steps), int(a.shape[0]), _ptr(a, C.c_int32), _ptr(s, C.c_int32),
                                C.c_uint64(seed), C.byref(out)))
        return out.value
    finally:
        if tmp is not None:
            os.unlink(path)


# ---- the benchmark workload, generated without the product library ----
STRESS_LIB = HERE / "_ref" / "libzsim_stress.so"
_stress = None


class StressConfigC(C.Structure):
    """zsim_stress_config (include/zsim_gpu.h)."""
    _fields_ = [("count", C.c_int32), ("num_steps", C.c_int32), ("agents", C.c_int32),
                ("road_points", C.c_int32), ("lanes", C.c_int32), ("lane_vertices", C.c_int32),
                ("dt", C.c_double), ("speed_limit", C.c_double), ("lane_width", C.c_double),
                ("first_index", C.c_int32), ("flags", C.c_int32)]


def _stress_lib() -> C.CDLL:
    global _stress
    if _stress is None:
        if not STRESS_LIB.exists():
            raise FileNotFoundError(f"{STRESS_LIB} not built (run oracle/build_oracle.py)")
        _stress = C.CDLL(str(STRESS_LIB))
        _stress.zstress_last_error.restype = C.c_char_p
        _stress.zstress_generate.argtypes = [C.POINTER(StressConfigC), C.c_uint64, C.POINTER(C.c_void_p),
                                             C.POINTER(C.c_size_t)]
        _stress.zstress_controlled_expand.argtypes = [C.c_void_p, C.c_size_t, C.c_double, C.c_double, C.c_double,
                                                      C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]
        _stress.zstress_free.argtypes = [C.c_void_p]
    return _stress


def _take(p: C.c_void_p, n: C.c_size_t) -> bytes:
    try:
        return np.ctypeslib.as_array((C.c_uint8 * n.value).from_address(p.value)).tobytes() if n.value else b""
    finally:
        _stress_lib().zstress_free(p)


def stress(count: int, agents: int, road_points: int, seed: int = 7, first_index: int = 0, c2: bool = False,
           num_steps: int = 92, lanes: int = 4, lane_vertices: int = 64) -> bytes:
    """ZSIM image of the stress scenarios [first_index, first_index + count)
    (the same bytes the product's ``stress_scenarios`` produces)."""
    L = _stress_lib()
    cfg = StressConfigC(count=count, num_steps=num_steps, agents=agents, road_points=road_points, lanes=lanes,
                        lane_vertices=lane_vertices, dt=0.1, speed_limit=10.0, lane_width=3.5,
                        first_index=first_index, flags=1 if c2 else 0)
    p, n = C.c_void_p(), C.c_size_t()
    rc = L.zstress_generate(C.byref(cfg), C.c_uint64(seed), C.byref(p), C.byref(n))
    if rc:
        raise RefError(rc, L.zstress_last_error().decode(errors="replace"))
    return _take(p, n)


def controlled_expand(zsim: bytes, config=None) -> bytes:
    """Per-row scenarios of every controllable actor (C2)."""
    L = _stress_lib()
    c = config_c(config)
    buf = C.create_string_buffer(bytes(zsim), len(zsim))
    p, n = C.c_void_p(), C.c_size_t()
    rc = L.zstress_controlled_expand(C.cast(buf, C.c_void_p), len(zsim), c.ego_length, c.ego_width,
                                     c.ego_center_offset, C.byref(p), C.byref(n))
    if rc:
        raise RefError(rc, L.zstress_last_error().decode(errors="replace"))
    return _take(p, n)


# ---- the reference's policy (core/nn/model.hpp, core/train/policy.hpp; ref_policy_shim.cpp) ----
class ModelConfigC(C.Structure):
    """zsim_model_config (include/zsim_gpu.h)."""
    _fields_ = [(n, C.c_int32) for n in ("latent", "heads", "trunk_blocks", "value_embed", "n_agents", "n_road",
                                          "n_route", "n_accel", "n_steer", "reserved")]


_PSIGS = {
    "zref_policy_last_error": (C.c_char_p, []),
    "zref_policy_param_count": (C.c_int, [C.POINTER(ModelConfigC), C.POINTER(C.c_int64)]),
    "zref_policy_init": (C.c_int, [C.POINTER(ModelConfigC), C.c_uint64, C.POINTER(C.c_float), C.c_int64]),
    "zref_policy_forward": (C.c_int, [C.POINTER(ModelConfigC), C.POINTER(C.c_float), C.c_int64, C.POINTER(ObsView),
                                      C.c_int32, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "zref_policy_act": (C.c_int, [C.POINTER(ModelConfigC), C.POINTER(C.c_float), C.c_int64, C.POINTER(ObsView),
                                  C.c_int32, C.c_int32, C.POINTER(C.c_uint64), C.POINTER(C.c_int32),
                                  C.POINTER(C.c_int32), C.POINTER(C.c_float), C.POINTER(C.c_float)]),
}


def _plib():
    L = lib()
    if not getattr(L, "_zref_policy_bound", False):
        for n, (r, a) in _PSIGS.items():
            f = getattr(L, n)
            f.restype = r
            f.argtypes = a
        L._zref_policy_bound = True
    return L


def _pcheck(code: int) -> None:
    if code != 0:
        raise RefError(code, _plib().zref_policy_last_error().decode(errors="replace"))


def model_config_c(cfg=None) -> ModelConfigC:
    """ModelConfig defaults (model.hpp:20-27); `cfg` any object with those attributes."""
    d = dict(latent=128, heads=2, trunk_blocks=2, value_embed=32, n_agents=16, n_road=128, n_route=64, n_accel=7,
             n_steer=5)
    return ModelConfigC(**{k: int(getattr(cfg, k, v)) for k, v in d.items()}, reserved=0)


def _obs_view(obs: dict, B: int):
    arrs = {k: np.ascontiguousarray(obs[k], dtype=np.float32) for k in ("active", "agents", "road", "route",
                                                                        "value_only")}
    v = ObsView(*[_ptr(arrs[k], C.c_float) for k in ("active", "agents", "road", "route", "value_only")])
    return v, arrs


def policy_param_count(cfg=None) -> int:
    n = C.c_int64()
    _pcheck(_plib().zref_policy_param_count(C.byref(model_config_c(cfg)), C.byref(n)))
    return n.value


def policy_init(cfg=None, seed: int = 0) -> np.ndarray:
    """Model<float>::make + init(seed) (model.hpp:174-216) in the reference."""
    n = policy_param_count(cfg)
    out = np.zeros(n, np.float32)
    _pcheck(_plib().zref_policy_init(C.byref(model_config_c(cfg)), C.c_uint64(seed), _ptr(out, C.c_float), n))
    return out


def policy_forward(params, obs: dict, B: int, cfg=None, double: bool = False):
    """The reference forward_row over B rows: (logits [B][n_accel+n_steer], value [B]),
    computed in Model<float> (the reference's arithmetic) or Model<double>."""
    c = model_config_c(cfg)
    p = np.ascontiguousarray(params, np.float32)
    v, keep = _obs_view(obs, B)
    logits = np.zeros((B, c.n_accel + c.n_steer))
    value = np.zeros(B)
    _pcheck(_plib().zref_policy_forward(C.byref(c), _ptr(p, C.c_float), p.size, C.byref(v), int(B), int(bool(double)),
                                        _ptr(logits, C.c_double), _ptr(value, C.c_double)))
    return logits, value


def policy_act(params, obs: dict, B: int, rng, use_argmax: bool, cfg=None) -> dict:
    """train::NNPolicy::act (policy.hpp:27-58) in the reference, one thread."""
    c = model_config_c(cfg)
    p = np.ascontiguousarray(params, np.float32)
    v, keep = _obs_view(obs, B)
    r = np.ascontiguousarray(rng, np.uint64).copy()
    out = dict(accel=np.zeros(B, np.int32), steer=np.zeros(B, np.int32), logp=np.zeros(B, np.float32),
               value=np.zeros(B, np.float32))
    _pcheck(_plib().zref_policy_act(C.byref(c), _ptr(p, C.c_float), p.size, C.byref(v), int(B), int(bool(use_argmax)),
                                    _ptr(r, C.c_uint64), _ptr(out["accel"], C.c_int32), _ptr(out["steer"], C.c_int32),
                                    _ptr(out["logp"], C.c_float), _ptr(out["value"], C.c_float)))
    out["rng"] = r
    return out


def bench_step(zsim, batch_sizes, steps: int, warmup: int, config=None) -> str:
    """The reference's own sim::bench_step (simcore.cpp:654-699): step-only
    timing at each batch size, zero actions, dones off -> bench_csv's CSV
    (batch_size,mean_step_ms,amortized_us_per_scenario)."""
    path, tmp = _as_path(zsim)
    try:
        bs = np.ascontiguousarray(batch_sizes, dtype=np.int32)
        ms = np.zeros(bs.size)
        cfg = config_c(config)
        _check(lib().zref_bench_step(path.encode(), _ptr(bs, C.c_int32), int(bs.size), int(steps), int(warmup),
                                     C.byref(cfg), _ptr(ms, C.c_double)))
        lines = ["batch_size,mean_step_ms,amortized_us_per_scenario"]
        lines += [f"{int(b)},{m:.6g},{m * 1000.0 / b:.6g}" for b, m in zip(bs, ms)]
        return "\n".join(lines) + "\n"
    finally:
        if tmp is not None:
            os.unlink(path)

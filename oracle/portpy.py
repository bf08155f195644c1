"""TEST INFRASTRUCTURE: Python handle on the plain-C restatement oracle
(oracle/zsim_oracle.c -> oracle/_build/libzsim_oracle.so).  Same surface as
oracle.refpy.RefEnv; builds the library on first use (gcc only).  Never
imported by the product path."""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from oracle.hostio import Obs, ObsView, OracleConfig, Out, SimConfigC, State, StateView, StepOutView, config_c
from oracle.hostio import ptr as _ptr
from oracle.hostio import state_view

HERE = Path(__file__).resolve().parent

_P = C.c_void_p
_SIGS = {
    "zor_last_error": (C.c_char_p, []),
    "zor_env_create": (C.c_int, [_P, C.c_size_t, C.POINTER(C.c_int64), C.c_int32, C.c_int32, C.POINTER(SimConfigC),
                                 C.POINTER(_P)]),
    "zor_env_destroy": (None, [_P]),
    "zor_env_info": (C.c_int, [_P, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "zor_scalars": (C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "zor_init_state": (C.c_int, [_P, C.c_uint64, C.POINTER(StateView)]),
    "zor_step": (C.c_int, [_P, C.POINTER(StateView), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                           C.POINTER(StateView), C.POINTER(StepOutView)]),
    "zor_observe": (C.c_int, [_P, C.POINTER(StateView), C.POINTER(ObsView), C.POINTER(C.c_int32)]),
}
_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        from oracle import build_oracle
        path = build_oracle.build_port()
        if path is None or not path.exists():
            raise FileNotFoundError("oracle/zsim_oracle.c could not be built")
        _lib = C.CDLL(str(path))
        for n, (r, a) in _SIGS.items():
            f = getattr(_lib, n)
            f.restype = r
            f.argtypes = a
    return _lib


class PortError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def _check(code: int) -> None:
    if code != 0:
        raise PortError(code, lib().zor_last_error().decode(errors="replace"))


class PortEnv:
    """C restatement of zsim::sim::Env over a ZSIM image."""

    def __init__(self, zsim, indices=None, horizon: int = 0, config=None):
        if isinstance(zsim, (str, Path)):
            zsim = Path(zsim).read_bytes()
        self._buf = C.create_string_buffer(bytes(zsim), len(zsim))
        self._config = config or OracleConfig()
        cfg = config_c(self._config)
        idx, n = None, 0
        if indices is not None:
            self._idx = np.ascontiguousarray(np.asarray(indices, dtype=np.int64))
            idx, n = self._idx.ctypes.data_as(C.POINTER(C.c_int64)), int(self._idx.size)
        h = C.c_void_p()
        _check(lib().zor_env_create(C.cast(self._buf, C.c_void_p), len(zsim), idx, n, int(horizon), C.byref(cfg),
                                    C.byref(h)))
        self.handle = h.value
        b, hz, ts = C.c_int32(), C.c_int32(), C.c_int32()
        _check(lib().zor_env_info(self.handle, C.byref(b), C.byref(hz), C.byref(ts)))
        self.batch, self.horizon, self.total_stop_lines = b.value, hz.value, ts.value

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                lib().zor_env_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    def batch_size(self) -> int:
        return self.batch

    def scalars(self):
        g, i, l = np.zeros(self.batch), np.zeros(self.batch), np.zeros(self.batch)
        _check(lib().zor_scalars(self.handle, _ptr(g, C.c_double), _ptr(i, C.c_double), _ptr(l, C.c_double)))
        return g, i, l

    def init_state(self, seed: int) -> State:
        st = State(self.batch, self.total_stop_lines)
        v = state_view(st)
        _check(lib().zor_init_state(self.handle, C.c_uint64(seed), C.byref(v)))
        return st

    def step(self, state: State, accel, steer):
        a = np.ascontiguousarray(accel, dtype=np.int32)
        s = np.ascontiguousarray(steer, dtype=np.int32)
        nxt, so = State(self.batch, self.total_stop_lines), Out(self.batch)
        vi, vo, vs = state_view(state), nxt.view(), so.view()
        _check(lib().zor_step(self.handle, C.byref(vi), _ptr(a, C.c_int32), _ptr(s, C.c_int32), C.byref(vo),
                              C.byref(vs)))
        return nxt, so

    def observe(self, state: State, with_topk: bool = False):
        c = self._config
        ob = Obs(self.batch, c.n_agents, c.n_road, c.n_route)
        tk = np.full((self.batch, c.n_agents + c.n_road + c.n_route), -1, np.int32)
        vi, vo = state_view(state), ob.view()
        _check(lib().zor_observe(self.handle, C.byref(vi), C.byref(vo), _ptr(tk, C.c_int32)))
        return (ob, tk) if with_topk else ob

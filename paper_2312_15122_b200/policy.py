"""Host-side mirror of the reference's policy objects on the device policy
kernels (include/zsim_gpu.h, zsim_policy_*):

  ModelConfig    nn/model.hpp:20-36
  Model.init     nn/model.hpp:199-212 (bit-exact, on the host)
  NNPolicy.act   train/policy.hpp:19-58, on device observation buffers

No CPU fallback: every call goes through libzsim_gpu.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._abi import ModelConfigC, ObsView, check, lib
from .env import DeviceObs, _stream


@dataclass
class ModelConfig:
    """ModelConfig (nn/model.hpp:20-27) with its ObsSpec (simcore.hpp:60-63)."""
    latent: int = 128
    heads: int = 2
    trunk_blocks: int = 2
    value_embed: int = 32
    n_agents: int = 16
    n_road: int = 128
    n_route: int = 64
    n_accel: int = 7
    n_steer: int = 5

    def to_c(self) -> ModelConfigC:
        return ModelConfigC(self.latent, self.heads, self.trunk_blocks, self.value_embed, self.n_agents,
                            self.n_road, self.n_route, self.n_accel, self.n_steer, 0)

    def param_count(self) -> int:
        n = C.c_int64()
        check(lib.zsim_policy_param_count(C.byref(self.to_c()), C.byref(n)))
        return n.value


def init_params(cfg: ModelConfig, seed: int) -> np.ndarray:
    """Model::init(seed) (nn/model.hpp:199-212): the flat float32 parameters."""
    out = np.zeros(cfg.param_count(), np.float32)
    check(lib.zsim_policy_init_params(C.byref(cfg.to_c()), C.c_uint64(seed),
                                      out.ctypes.data_as(C.POINTER(C.c_float)), out.size))
    return out


class NNPolicy:
    """NNPolicy (train/policy.hpp:19-58) over device observation buffers.

    `act_device` mirrors NNPolicy::act: per row, forward_row then argmax
    (use_argmax) or sample_categorical on each head with the row's rng
    stream, advanced in place.  All pointers are device addresses (ints)."""

    PRECISIONS = {"tf32": 0, "fp32": 1}

    def __init__(self, cfg: ModelConfig, params: np.ndarray, use_argmax: bool = False, device: int = 0,
                 precision: str = "fp32"):
        """precision "fp32" (default): every contraction on the FP32 pipe, the
        reference's Model<float> arithmetic; "tf32": the projections on the
        tcgen05 tensor cores (tf32 inputs, fp32 accumulate) -- faster, with
        logits ~1e-4 from fp32, so sampled / argmax actions can differ where
        the decision margin is that small."""
        self.cfg = cfg
        self.argmax = bool(use_argmax)
        p = np.ascontiguousarray(params, np.float32)
        h = C.c_void_p()
        check(lib.zsim_policy_create(C.byref(cfg.to_c()), p.ctypes.data_as(C.POINTER(C.c_float)), p.size, device,
                                     C.byref(h)))
        self._h = h
        self.precision = precision
        check(lib.zsim_policy_set_precision(h, self.PRECISIONS[precision]))

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def close(self):
        if self._h:
            lib.zsim_policy_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def act_device(self, obs: DeviceObs | ObsView, batch: int, rng_ptr: int, accel_ptr: int, steer_ptr: int, logp_ptr: int,
                   value_ptr: int, logits_ptr: int = 0, stream=None) -> None:
        view = obs.v if isinstance(obs, DeviceObs) else obs
        check(lib.zsim_policy_act(self._h, C.byref(view), int(batch), C.c_void_p(rng_ptr or None),
                                  int(self.argmax), C.c_void_p(accel_ptr), C.c_void_p(steer_ptr),
                                  C.c_void_p(logp_ptr), C.c_void_p(value_ptr), C.c_void_p(logits_ptr or None),
                                  _stream(stream)))

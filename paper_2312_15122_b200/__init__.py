"""B200-native batched driving-simulator step (arXiv 2312.15122 reference path).

The product is the native library ``libzsim_gpu.so`` (sm_100a kernels behind
the C-ABI of ``include/zsim_gpu.h``); this package is its host-side mirror of
the reference's ``zsim::sim::Env`` API.  Importing it loads the native library
and fails loudly when it is missing -- there is no CPU fallback.
"""
from ._abi import ZsimError, lib  # noqa: F401
from .env import (AGGREGATE_FIELDS, DONE_REASONS, BatchStream, DeviceEpisode, DeviceObs, DeviceState, DeviceStepOut,  # noqa: F401
                  Env, ObservationBatch, aggregate_finalize,
                  STRESS_C2, SimConfig, SimStateBatch, StepOut, StressConfig, controlled_expand, event_bit,
                  random_actions, stress_scenarios)
from .policy import ModelConfig, NNPolicy, init_params  # noqa: F401
from .config import KeyValue, sim_config_from_kv, sim_config_to_kv  # noqa: F401

__all__ = ["Env", "SimConfig", "SimStateBatch", "StepOut", "ObservationBatch", "DeviceState", "DeviceStepOut",
           "DeviceObs", "StressConfig", "stress_scenarios", "random_actions", "ZsimError", "DONE_REASONS",
           "event_bit", "lib", "controlled_expand", "STRESS_C2", "DeviceEpisode", "aggregate_finalize",
           "AGGREGATE_FIELDS", "BatchStream", "ModelConfig", "NNPolicy", "init_params", "KeyValue",
           "sim_config_from_kv", "sim_config_to_kv"]

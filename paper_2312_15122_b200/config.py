"""Flat ``key = value`` configs (the reference's ``cfg::KeyValue``,
core/config.hpp:13-43, config.cpp:22-129) for ``SimConfig`` and the benchmark
workload, with the same dump and FNV-1a hash, so every result JSON can carry
the hash of the configuration it ran ("Config / flags").

Semantics follow the reference: ``#`` starts a comment; keys and values are
trimmed; a later duplicate key wins; keys are kept sorted so ``dump()`` and
``hash()`` do not depend on input order; numbers set from Python doubles are
written with 17 significant digits (``ostream::precision(17)``); every
``get_*`` marks its key used and ``unused_keys()`` lists the rest (strict
loading rejects unknown keys).
"""
from __future__ import annotations

import re
from dataclasses import fields

from ._abi import ZsimError

_CONFIG = 2  # ErrorKind::config
_INT_RE = re.compile(r"-?[0-9]+", re.ASCII)


def fnv1a(data: bytes, h: int = 0xCBF29CE484222325) -> int:
    """FNV-1a 64 (common.hpp:62-69)."""
    for b in data:
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def _fmt_double(v: float) -> str:
    """ostream << double at precision(17) (config.cpp:108-113): %.17g."""
    return format(float(v), ".17g")


class KeyValue:
    """cfg::KeyValue (config.hpp:13-43)."""

    def __init__(self):
        self._values: dict[str, str] = {}
        self._touched: set[str] = set()

    @classmethod
    def parse_text(cls, text: str, origin: str = "<memory>") -> "KeyValue":
        kv = cls()
        for lineno, line in enumerate(text.split("\n"), 1):
            hp = line.find("#")
            if hp >= 0:
                line = line[:hp]
            line = line.strip(" \t\r\n")
            if not line:
                continue
            eq = line.find("=")
            if eq < 0:
                raise ZsimError(_CONFIG, f"{origin}:{lineno}: expected `key = value`")
            key, value = line[:eq].strip(" \t\r\n"), line[eq + 1:].strip(" \t\r\n")
            if not key:
                raise ZsimError(_CONFIG, f"{origin}:{lineno}: empty key")
            kv._values[key] = value
        return kv

    @classmethod
    def parse_file(cls, path) -> "KeyValue":
        try:
            with open(path) as f:
                text = f.read()
        except OSError:
            raise ZsimError(3, f"cannot open config file: {path}") from None
        return cls.parse_text(text, str(path))

    def has(self, key: str) -> bool:
        return key in self._values

    def get_string(self, key: str, fallback: str) -> str:
        self._touched.add(key)
        return self._values.get(key, fallback)

    def get_double(self, key: str, fallback: float) -> float:
        self._touched.add(key)
        if key not in self._values:
            return fallback
        v = self._values[key]
        try:
            if "_" in v or not v:  # std::stod must consume the whole value
                raise ValueError(v)
            return float(v)
        except ValueError:
            raise ZsimError(_CONFIG, f"config key `{key}`: not a number: {v}") from None

    def get_int(self, key: str, fallback: int) -> int:
        self._touched.add(key)
        if key not in self._values:
            return fallback
        v = self._values[key]
        try:
            if not _INT_RE.fullmatch(v):  # std::from_chars, base 10
                raise ValueError(v)
            return int(v, 10)
        except ValueError:
            raise ZsimError(_CONFIG, f"config key `{key}`: not an integer: {v}") from None

    def get_bool(self, key: str, fallback: bool) -> bool:
        self._touched.add(key)
        if key not in self._values:
            return fallback
        v = self._values[key]
        if v in ("true", "1", "yes", "on"):
            return True
        if v in ("false", "0", "no", "off"):
            return False
        raise ZsimError(_CONFIG, f"config key `{key}`: not a boolean: {v}")

    def set(self, key: str, value) -> None:
        if isinstance(value, bool):
            value = int(value)
        if isinstance(value, int):
            self._values[key] = str(value)
        elif isinstance(value, float):
            self._values[key] = _fmt_double(value)
        else:
            self._values[key] = str(value)

    def unused_keys(self) -> list[str]:
        return [k for k in sorted(self._values) if k not in self._touched]

    def dump(self) -> str:
        return "".join(f"{k} = {self._values[k]}\n" for k in sorted(self._values, key=lambda s: s.encode()))

    def hash(self) -> int:
        return fnv1a(self.dump().encode())


_INT_FIELDS = ("n_agents", "n_road", "n_route", "threads")


def sim_config_to_kv(cfg) -> KeyValue:
    """SimConfig (simcore.hpp:14-45) as a KeyValue, keys = field names."""
    kv = KeyValue()
    for f in fields(cfg):
        v = getattr(cfg, f.name)
        kv.set(f.name, int(v) if f.name in _INT_FIELDS or f.name == "disable_dones" else float(v))
    return kv


def sim_config_from_kv(kv: KeyValue, strict: bool = True):
    """SimConfig from a KeyValue (missing keys keep the defaults); `strict`
    rejects keys that are not SimConfig fields."""
    from .env import SimConfig
    cfg = SimConfig()
    for f in fields(cfg):
        d = getattr(cfg, f.name)
        if f.name == "disable_dones":
            setattr(cfg, f.name, kv.get_bool(f.name, bool(d)))
        elif f.name in _INT_FIELDS:
            setattr(cfg, f.name, kv.get_int(f.name, int(d)))
        else:
            setattr(cfg, f.name, kv.get_double(f.name, float(d)))
    if strict and kv.unused_keys():
        raise ZsimError(_CONFIG, f"unknown SimConfig keys: {', '.join(kv.unused_keys())}")
    return cfg

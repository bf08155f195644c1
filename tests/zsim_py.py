"""Pure-Python reader of the ZSIM container (scenario.hpp:97-104,
scenario_io.cpp:132-189) for tests: lets the parity suite look at raw
scenario arrays (road points, agents) independently of either implementation."""
from __future__ import annotations

import struct

import numpy as np


class _R:
    def __init__(self, b: bytes, off: int):
        self.b, self.o = b, off

    def u8(self):
        v = self.b[self.o]
        self.o += 1
        return v

    def u32(self):
        v = struct.unpack_from("<I", self.b, self.o)[0]
        self.o += 4
        return v

    def f32(self):
        v = struct.unpack_from("<f", self.b, self.o)[0]
        self.o += 4
        return v

    def s(self):
        n = self.u32()
        v = self.b[self.o:self.o + n].decode()
        self.o += n
        return v

    def f32s(self):
        n = self.u32()
        v = np.frombuffer(self.b, dtype="<f4", count=n, offset=self.o).copy()
        self.o += 4 * n
        return v

    def u8s(self):
        n = self.u32()
        v = np.frombuffer(self.b, dtype=np.uint8, count=n, offset=self.o).copy()
        self.o += n
        return v


def read_zsim(b: bytes) -> list[dict]:
    assert b[:4] == b"ZSIM"
    version, _ = struct.unpack_from("<HH", b, 4)
    assert version == 1
    dt = struct.unpack_from("<d", b, 8)[0]
    off = 16
    out = []
    while off < len(b):
        n = struct.unpack_from("<I", b, off)[0]
        r = _R(b, off + 4)
        sc = {"dt": dt, "id": r.s(), "num_steps": r.u32()}
        sc["ego"] = {k: r.f32s() for k in ("x", "y", "heading", "v")}
        sc["agents"] = []
        for _ in range(r.u32()):
            a = {"id": r.s(), "length": r.f32(), "width": r.f32()}
            for k in ("x", "y", "heading", "speed"):
                a[k] = r.f32s()
            a["valid"] = r.u8s()
            sc["agents"].append(a)
        sc["lanes"] = []
        for _ in range(r.u32()):
            sc["lanes"].append({"lane_id": r.u32(), "left": r.f32s(), "right": r.f32s(), "s_start": r.f32(),
                                "s_end": r.f32()})
        sc["features"] = []
        for _ in range(r.u32()):
            k, d = r.u8(), r.u8()
            sc["features"].append({"kind": k, "dir": d, "xy": r.f32s()})
        sc["lights"] = []
        for _ in range(r.u32()):
            sc["lights"].append({"signal_id": r.u32(), "stop_x": r.f32(), "stop_y": r.f32(), "state": r.u8s()})
        sc["stops"] = []
        for _ in range(r.u32()):
            sc["stops"].append({"xy": r.f32s(), "pos_x": r.f32(), "pos_y": r.f32()})
        sc["speed_limit"], sc["goal_x"], sc["goal_y"] = r.f32(), r.f32(), r.f32()
        assert r.o == off + 4 + n, "record length mismatch"
        out.append(sc)
        off += 4 + n
    return out


def _p_str(o: bytearray, s: str) -> None:
    b = s.encode()
    o += struct.pack("<I", len(b)) + b


def _p_f32s(o: bytearray, a) -> None:
    a = np.asarray(a, dtype="<f4")
    o += struct.pack("<I", a.size) + a.tobytes()


def _p_u8s(o: bytearray, a) -> None:
    a = np.asarray(a, dtype=np.uint8)
    o += struct.pack("<I", a.size) + a.tobytes()


def write_zsim(scenarios: list[dict], dt: float = 0.1) -> bytes:
    """Inverse of read_zsim (encode_record, scenario_io.cpp:80-130)."""
    out = bytearray(b"ZSIM" + struct.pack("<HHd", 1, 0, dt))
    for sc in scenarios:
        r = bytearray()
        _p_str(r, sc.get("id", "s"))
        r += struct.pack("<I", sc["num_steps"])
        for k in ("x", "y", "heading", "v"):
            _p_f32s(r, sc["ego"][k])
        r += struct.pack("<I", len(sc["agents"]))
        for a in sc["agents"]:
            _p_str(r, a.get("id", "a"))
            r += struct.pack("<ff", a["length"], a["width"])
            for k in ("x", "y", "heading", "speed"):
                _p_f32s(r, a[k])
            _p_u8s(r, a["valid"])
        r += struct.pack("<I", len(sc["lanes"]))
        for l in sc["lanes"]:
            r += struct.pack("<I", l["lane_id"])
            _p_f32s(r, l["left"])
            _p_f32s(r, l["right"])
            r += struct.pack("<ff", l["s_start"], l["s_end"])
        r += struct.pack("<I", len(sc["features"]))
        for f in sc["features"]:
            r += struct.pack("<BB", f["kind"], f["dir"])
            _p_f32s(r, f["xy"])
        r += struct.pack("<I", len(sc["lights"]))
        for t in sc["lights"]:
            r += struct.pack("<Iff", t.get("signal_id", 1), t["stop_x"], t["stop_y"])
            _p_u8s(r, t["state"])
        r += struct.pack("<I", len(sc["stops"]))
        for s_ in sc["stops"]:
            _p_f32s(r, s_["xy"])
            r += struct.pack("<ff", s_["pos_x"], s_["pos_y"])
        r += struct.pack("<fff", sc["speed_limit"], sc["goal_x"], sc["goal_y"])
        out += struct.pack("<I", len(r)) + r
    return bytes(out)


def straight_scenario(n: int = 20, v: float = 10.0, heading: float = 0.0, length: float = 200.0, agents=(),
                      lights=(), stops=(), goal=None, features=None, limit: float = 10.0) -> dict:
    """A straight single-lane route along +x (lane width 3.5 m) with the ego
    logged at constant speed from the origin; helpers for SPEC known-answer
    tests.  `agents` are dicts with x/y/heading/length/width (static)."""
    xs = np.arange(0.0, length + 1e-9, 2.0)
    ego_x = np.array([v * 0.1 * t * np.cos(heading) for t in range(n)])
    ego_y = np.array([v * 0.1 * t * np.sin(heading) for t in range(n)])
    sc = {"id": "kat", "num_steps": n,
          "ego": {"x": ego_x, "y": ego_y, "heading": np.full(n, heading), "v": np.full(n, v)},
          "agents": [], "lanes": [{"lane_id": 0, "left": np.stack([xs, np.full_like(xs, 1.75)], 1).ravel(),
                                    "right": np.stack([xs, np.full_like(xs, -1.75)], 1).ravel(),
                                    "s_start": 0.0, "s_end": float(length)}],
          "features": features if features is not None else [
              {"kind": 0, "dir": 1, "xy": np.stack([xs, np.full_like(xs, 1.75)], 1).ravel()}],
          "lights": list(lights), "stops": list(stops), "speed_limit": limit,
          "goal_x": float(goal[0]) if goal else float(length - 10), "goal_y": float(goal[1]) if goal else 0.0}
    for a in agents:
        sc["agents"].append({"id": "a", "length": a.get("length", 4.0), "width": a.get("width", 2.0),
                             "x": np.full(n, a["x"]), "y": np.full(n, a["y"]),
                             "heading": np.full(n, a.get("heading", 0.0)), "speed": np.full(n, a.get("speed", 0.0)),
                             "valid": np.ones(n, np.uint8)})
    return sc

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

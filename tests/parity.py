"""Parity comparison helpers (test infrastructure).

Tolerances are the north-star contract (BASELINE.json): fp outputs within
1e-5 relative / 1e-6 absolute; flags, reasons, events, done, top-k membership
and slot validity bit-exact.  Top-k slot lists are compared slot by slot;
where two candidates' sort keys are equal (or equal up to the last-ulp
differences between device and glibc trig), the slots are compared as a
multiset within that tie group for ROAD slots only -- the reference orders road
points by d2 only (roads.cpp:231-232), so its order inside exact ties is
libstdc++-defined.  Agent and route slots are ordered by (key, index) in the
reference and must match slot by slot.
"""
from __future__ import annotations

import numpy as np

RTOL = 1e-5
ATOL = 1e-6

STATE_EXACT = ("t", "done", "reason", "rng", "proj_in_corridor", "events", "stopped_flags")
STATE_TOL = ("x", "y", "heading", "v", "steering", "proj_s", "proj_d")
STEPOUT_EXACT = ("event",)
STEPOUT_TOL = ("reward", "s", "a_lat", "a_lon", "v")


def close(a, b, rtol=RTOL, atol=ATOL):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.abs(a - b) <= atol + rtol * np.abs(b)


def compare_state(g, r, tag="") -> list[str]:
    errs = []
    for f in STATE_EXACT:
        a, b = getattr(g, f), getattr(r, f)
        if not np.array_equal(a, b):
            bad = np.nonzero(a != b)[0]
            errs.append(f"{tag}state.{f} differs at rows {bad[:8].tolist()} (gpu {a[bad[:4]]} ref {b[bad[:4]]})")
    for f in STATE_TOL:
        a, b = getattr(g, f), getattr(r, f)
        ok = close(a, b)
        if not ok.all():
            bad = np.nonzero(~ok)[0]
            errs.append(f"{tag}state.{f} out of tol at rows {bad[:8].tolist()} (gpu {a[bad[:3]]} ref {b[bad[:3]]})")
    return errs


def compare_stepout(g, r, tag="") -> list[str]:
    errs = []
    for f in STEPOUT_EXACT:
        a, b = getattr(g, f), getattr(r, f)
        if not np.array_equal(a, b):
            bad = np.nonzero(a != b)[0]
            errs.append(f"{tag}stepout.{f} differs at rows {bad[:8].tolist()}")
    for f in STEPOUT_TOL:
        a, b = getattr(g, f), getattr(r, f)
        ok = close(a, b)
        if not ok.all():
            bad = np.nonzero(~ok)[0]
            errs.append(f"{tag}stepout.{f} out of tol at rows {bad[:8].tolist()} (gpu {a[bad[:3]]} ref {b[bad[:3]]})")
    return errs


def _slot_key(rows: np.ndarray, kind: str) -> np.ndarray:
    if kind == "agents":
        return rows[:, 4].astype(np.float64)  # bbox distance (simcore.cpp:472-474)
    x = rows[:, 0].astype(np.float64)
    y = rows[:, 1].astype(np.float64)
    return x * x + y * y  # rotation preserves the d2 sort key (roads.cpp:231, simcore.cpp:517)


def compare_slots(g: np.ndarray, r: np.ndarray, kind: str, valid_col: int, exact_cols) -> str | None:
    """One row's slot list [K][F]; returns None when equivalent."""
    vg, vr = g[:, valid_col], r[:, valid_col]
    if not np.array_equal(vg, vr):
        return f"valid pattern differs ({int(vg.sum())} vs {int(vr.sum())} slots)"
    n = int(vr.sum())
    if n == 0:
        return None if np.array_equal(g, r) else "empty rows not zero"
    if not np.array_equal(g[n:], r[n:]):
        return "padding slots not zero"
    G, R = g[:n].astype(np.float64), r[:n].astype(np.float64)

    def rows_match(a, b):
        return bool(close(a, b).all() and np.array_equal(a[:, exact_cols], b[:, exact_cols]))

    if rows_match(G, R):
        return None
    if kind != "road":
        # agents (simcore.cpp:472-474) and route (:517-519) sort by (key, index):
        # the order is deterministic, so slot i must match slot i.
        bad = np.nonzero(~np.array([rows_match(G[i:i + 1], R[i:i + 1]) for i in range(n)]))[0]
        return f"slot {int(bad[0])} differs (ordered by (key, index) in the reference)"
    # road: nearest_features sorts by d2 only (roads.cpp:231-232) -- inside a
    # group of equal keys the reference order is libstdc++-defined, so tie
    # groups compare as multisets
    kr = _slot_key(R, kind)
    kg = _slot_key(G, kind)
    if not close(kg, kr, rtol=1e-4, atol=1e-5).all():
        return "slot keys differ beyond tie tolerance"
    start = 0
    while start < n:
        end = start + 1
        while end < n and abs(kr[end] - kr[start]) <= 1e-5 * (1.0 + abs(kr[start])):
            end += 1
        a, b = G[start:end], R[start:end]
        if not rows_match(a, b):
            oa = np.lexsort(a.T[::-1])
            ob = np.lexsort(b.T[::-1])
            if not rows_match(a[oa], b[ob]):
                if end == n and n == g.shape[0]:
                    # tie group cut by k: which of the equal-key candidates fill
                    # the last slots is unspecified, but every member must carry
                    # the group's key and be a valid slot
                    if not close(np.sort(kg[start:end]), np.sort(kr[start:end]), rtol=1e-4, atol=1e-5).all():
                        return f"k-cut tie group {start}..{end - 1}: keys differ"
                else:
                    return f"slots {start}..{end - 1} differ (tie group of {end - start})"
        start = end
    return None


def compare_obs(g, r, tag="") -> list[str]:
    errs = []
    # active: v, steering, d_stop, light one-hot (exact), d_light, limit
    ok = close(g.active, r.active)
    if not ok.all():
        bad = np.nonzero(~ok.all(1))[0]
        errs.append(f"{tag}obs.active out of tol at rows {bad[:8].tolist()}")
    if not np.array_equal(g.active[:, 3:7], r.active[:, 3:7]):
        errs.append(f"{tag}obs.active light one-hot differs")
    if not close(g.value_only, r.value_only).all():
        errs.append(f"{tag}obs.value_only out of tol")
    specs = (("agents", 5, [5]), ("road", 11, list(range(2, 12))), ("route", 4, [2, 3, 4]))
    for name, vcol, exact in specs:
        G, R = getattr(g, name), getattr(r, name)
        for b in range(G.shape[0]):
            m = compare_slots(G[b], R[b], name, vcol, exact)
            if m:
                errs.append(f"{tag}obs.{name} row {b}: {m}")
                break
    return errs

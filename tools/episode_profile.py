"""Per-step cost profile of the fused kernel over one C1 episode.

    python tools/episode_profile.py [B]               # kernel time at each t (product library)
    ZSIM_GPU_LIB=paper_2312_15122_b200/_build/pathstats/libzsim_gpu_pathstats.so \\
        python tools/episode_profile.py [B] --pathstats   # + which top-k / agent paths each step took

Diagnostic tool, not the bench.  Prints one JSON object.
"""
import ctypes as C
import gc
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2312_15122_b200 as z
from paper_2312_15122_b200 import _abi

NAMES = ["rows_obs", "road_T_hint", "road_T_chunk", "road_T_none", "road_hist", "road_linear", "road_slow", "road_C",
         "road_nlist", "route_T_hint", "route_T_chunk", "route_T_none", "route_hist", "route_linear", "route_slow",
         "route_C", "route_nlist", "ag_surv", "ag_cand", "ag_cand_overflow", "ag_contact", "proj_extra", "proj_calls",
         "rows_step"]


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    B = int(args[0]) if args else 4096
    pathstats = "--pathstats" in sys.argv
    c2 = "--c2" in sys.argv  # C2 shapes: B scenarios x 128 controlled actors, 8k road points
    n_ag = int(next((a[9:] for a in sys.argv if a.startswith("--agents=")), "128" if c2 else "32"))
    zsim = z.stress_scenarios(z.StressConfig(count=B, agents=n_ag, road_points=8192 if c2 or n_ag > 32 else 2048,
                                             flags=z.STRESS_C2 if c2 else 0), 7)
    env = z.Env(zsim, config=z.SimConfig(disable_dones=True), controlled=c2)
    B = env.info.batch
    pol = next((int(a[9:]) for a in sys.argv if a.startswith("--policy=")), None)
    if pol is not None:
        env.set_launch_policy(pol)
    acc, st = z.random_actions(91, B, seed=123)
    dA, dS = torch.from_numpy(acc).cuda(), torch.from_numpy(st).cuda()
    s0, s1, so, ob = env.device_state(), env.device_state(), env.device_stepout(), env.device_obs()
    stream = torch.cuda.current_stream()
    fn = None
    buf = (C.c_ulonglong * 32)()
    if pathstats:
        lib = _abi.load_library()
        fn = lib.zsimdbg_pathstats
        fn.argtypes = [C.POINTER(C.c_ulonglong), C.c_int, C.c_void_p, C.c_int]
        fn.restype = C.c_int
    res = {"B": B, "ms": [], "stats": [], "phases": {}}
    cyc = np.zeros((B, 24), dtype=np.uint32)
    PH = ["project", "collide+flags", "active+agents", "road_topk", "road_feat", "route_topk", "route_feat"]
    gc.disable()
    for ep in range(int(next((a[5:] for a in sys.argv if a.startswith("--eps")), "2"))):  # episode 0 warms up
        env.reset_device(42, s0, stream)
        if fn:
            fn(buf, 1, None, 0)
        for t in range(91):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            if "--split" in sys.argv:  # separate step and observe kernels
                env.step_device(s0, dA[t].data_ptr(), dS[t].data_ptr(), s1, so, stream)
                env.observe_device(s1, ob, stream)
            else:
                env.step_observe_device(s0, dA[t].data_ptr(), dS[t].data_ptr(), s1, so, ob, stream)
            e1.record(stream)
            s0, s1 = s1, s0
            if "--sync" in sys.argv:
                torch.cuda.synchronize()
            if fn:
                torch.cuda.synchronize()
                fn(buf, 1, cyc.ctypes.data, B)
                if ep == 1:
                    res["stats"].append(list(buf)[:len(NAMES)])
                if ep == 1 and t in (5, 40, 80):
                    d = np.diff(cyc[:, :8].astype(np.int64), axis=1) % (1 << 32)  # [B][7]
                    seq = [0, 8, 9, 10, 11, 12, 13, 14, 15, 1]
                    sub = np.diff(cyc[:, seq].astype(np.int64), axis=1) % (1 << 32)
                    tot = d.sum(1)
                    slow = np.argsort(tot)[-max(1, B // 100):]
                    res["phases"][t] = {
                        "row_total": {"mean": float(tot.mean()), "p99": float(np.percentile(tot, 99)),
                                      "max": float(tot.max())},
                        "mean": dict(zip(PH, d.mean(0).round(0).tolist())),
                        "slowest_1pct_mean": dict(zip(PH, d[slow].mean(0).round(0).tolist())),
                        "project_split": dict(zip(["load+flags", "bicycle+queries", "groups", "fp32_pass", "thresholds",
                                                   "exact", "argmin", "lane_hit", "rest"], sub.mean(0).round(0).tolist())),
                        "project_split_slowest_1pct": dict(zip(["load+flags", "bicycle+queries", "groups", "fp32_pass",
                                                                "thresholds", "exact", "argmin", "lane_hit", "rest"],
                                                               sub[slow].mean(0).round(0).tolist())),
                        "agents_split": dict(zip(["active", "distances", "order", "features"],
                                                 (np.diff(cyc[:, [2, 16, 17, 18, 3]].astype(np.int64), axis=1)
                                                  % (1 << 32)).mean(0).round(0).tolist())),
                        "slowest_row": int(np.argmax(tot)), "slowest_row_phases": dict(zip(PH, d[np.argmax(tot)].tolist())),
                    }
            if ep >= 1:
                res["ms"].append((e0, e1))
        torch.cuda.synchronize()
    res["ms"] = [round(a.elapsed_time(b) * 1000, 1) for a, b in res["ms"]]
    if fn:
        tot = np.array(res["stats"], dtype=np.float64)
        res["totals"] = dict(zip(NAMES, tot.sum(0).tolist()))
        # per-step means normalised by rows, every 10th step
        res["per_t"] = {t: {n: round(v / max(1, tot[t][0]), 3) for n, v in zip(NAMES, tot[t])} for t in
                        range(0, 91, 10)}
        del res["stats"]
    print(json.dumps(res))


if __name__ == "__main__":
    main()

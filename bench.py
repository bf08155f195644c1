#!/usr/bin/env python
"""Throughput benchmark of the batched simulator step (BASELINE.json metric).

One "step" = one fused step+observe launch over the whole scenario batch
(Env::step then Env::observe of the stepped state, simcore.cpp:590-609).
Episodes are 91 steps long (T_log = 92); the state is re-initialised (reset
kernel, inside the timed region) every 91 steps.  Throughput runs use
`disable_dones = true` like the reference bench (simcore.cpp:669).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C1] [--impl ours|reference]

`--gpus N` without torchrun re-launches itself under torch.distributed.run
(one process per GPU, 127.0.0.1 rendezvous).  Each rank simulates its own
shard of scenarios; no data-path collective.  The only exchange is the
per-rollout episode-stats all-reduce over NCCL through the library's C-ABI
(zsim_stats_allreduce).  C1 / C2 are per-GPU workloads (weak
scaling); C3 / C4 are BASELINE's fixed global sets (65,536 and 131,072
scenarios) split across the ranks (strong scaling).  Rank 0 prints ONE JSON
line.  The timed region is exactly K launches (plus the resets at t % 91 == 0)
replayed from one CUDA graph.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import socket
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "simulated agent-steps/sec (device-timed) at 1/2/4/8 B200; % HBM roofline"
UNIT = "agent-steps/s"
EPISODE = 91  # steps per episode (92 logged states)
STRESS_SEED, ACTION_SEED, RESET_SEED = 7, 123, 42

# BASELINE.json configs.  `per_gpu`: scenarios each
# GPU simulates (weak scaling); `global`: one fixed set split over the GPUs.
CONFIGS = {
    "C0": dict(per_gpu=64, agents=32, road_points=2048,
               workload="C0: 64 scenarios x 32 agents, 2k roadgraph points, 91-step rollouts (CPU reference case)"),
    "C1": dict(per_gpu=4096, agents=32, road_points=2048,
               workload="C1: 1xB200, 4096 scenarios x 32 agents, 2k roadgraph points, top-k 16 agents / 128 "
                        "polyline pts"),
    "C2": dict(per_gpu=4096, agents=128, road_points=8192, controlled=True,
               workload="C2 dense: 4096 scenarios x 128 agents all controlled (524,288 ego rows), 8k roadgraph "
                        "points; agent-steps = controlled rows x steps (SURVEY 8a row 20)"),
    "C3": dict(global_=65536, agents=64, road_points=4096,
               workload="C3: 65536 scenarios x 64 agents, 4k roadgraph points, 91-step rollouts, scenario-sharded "
                        "over the GPUs"),
    "C4": dict(global_=131072, agents=128, road_points=8192,
               workload="C4: 131072 scenarios x 128 agents, 8k roadgraph points, scenario-sharded over the GPUs, "
                        "stats allreduce"),
    "C4s": dict(per_gpu=16384, agents=128, road_points=8192,
                workload="C4 per-GPU shard at 8 GPUs: 16384 scenarios x 128 agents, 8k roadgraph points"),
}
LANES, LANE_VERTICES = 4, 64


def scenario_step_bytes(A: int, P: int, R: int = 2 * LANES * LANE_VERTICES, L: int = LANES,
                        C: int = LANE_VERTICES) -> int:
    """Algorithmic HBM bytes per scenario-step of the fused step+observe
    (SURVEY.md §8d): reads state 80, actions 8, agent slices 38(A-1), road
    10P, route 10R, lane centerlines 32LC, lights/stops/goal 64; writes state
    80, StepOut 21, observation 7852."""
    return 80 + 8 + 38 * (A - 1) + 10 * P + 10 * R + 32 * L * C + 64 + 80 + 21 + 7852


def controlled_row_step_bytes(A: int, P: int, R: int = 2 * LANES * LANE_VERTICES, L: int = LANES,
                              C: int = LANE_VERTICES) -> float:
    """C2: the scenario's static data (agent slices of all A actors, road,
    route, lanes, lights/stops) is read once per scenario-step and shared by
    its A rows; each row reads state + actions and writes state, StepOut and
    its observation (~1.14 MB per scenario-step at A=128, P=8192)."""
    shared = 38 * A + 10 * P + 10 * R + 32 * L * C + 64
    return shared / A + 80 + 8 + 80 + 21 + 7852


def hbm_peak() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


def plan(name: str, world: int, override: int = 0) -> dict:
    """The job: global scenario count, scaling mode; identical in both arms."""
    c = dict(CONFIGS[name])
    strong = "global_" in c
    total = override or (c["global_"] if strong else c["per_gpu"] * world)
    c.update(name=name, total=total, scaling="strong" if strong else "weak", controlled=bool(c.get("controlled")))
    c["rows_per_scenario"] = c["agents"] if c["controlled"] else 1
    return c


# SimConfig of every run (simcore.hpp:14-45 defaults, dones off), as key = value
SIM_CONFIG = dict(wheelbase=3.0, ego_length=4.7, ego_width=1.9, ego_center_offset=1.5, delta_max=0.55, v_min=0.0,
                  goal_radius=2.0, footprint_margin=0.1, stop_cross_speed=0.5, stop_zone=2.0, stop_slow_speed=0.1,
                  disable_dones=1, w_progress=1.0, w_speed=0.1, w_lat=0.02, w_lon=0.02, terminal_penalty=10.0,
                  n_agents=16, n_road=128, n_route=64, feature_radius=100.0, threads=1)


def config_hash(p: dict) -> str:
    """FNV-1a of the run's flat `key = value` dump (the reference's
    cfg::KeyValue dump / hash, config.cpp:116-126; paper_2312_15122_b200.config):
    the workload keys plus the SimConfig, so every result JSON names the exact
    configuration it ran."""
    vals = {f"sim.{k}": (format(v, ".17g") if isinstance(v, float) else str(v)) for k, v in SIM_CONFIG.items()}
    vals.update({"bench.config": p["name"], "bench.scenarios": str(p["total"]), "bench.agents": str(p["agents"]),
                 "bench.road_points": str(p["road_points"]), "bench.controlled": str(int(p["controlled"])),
                 "bench.lanes": str(LANES), "bench.lane_vertices": str(LANE_VERTICES),
                 "bench.steps_per_episode": str(EPISODE), "bench.seed.scenarios": str(STRESS_SEED),
                 "bench.seed.actions": str(ACTION_SEED), "bench.seed.reset": str(RESET_SEED)})
    dump = "".join(f"{k} = {vals[k]}\n" for k in sorted(vals, key=lambda x: x.encode())).encode()
    h = 0xCBF29CE484222325
    for b in dump:
        h = ((h ^ b) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def config_block(p: dict, world: int) -> dict:
    """`config` of the JSON line -- the same keys and values in both arms."""
    return {"workload": p["workload"], "config_id": p["name"], "config_hash": config_hash(p), "scenarios": p["total"],
            "scenarios_per_gpu": -(-p["total"] // world), "agents": p["agents"], "road_points": p["road_points"],
            "controlled": p["controlled"], "rows": p["total"] * p["rows_per_scenario"],
            "route_points": 2 * LANES * LANE_VERTICES, "lanes": LANES, "lane_vertices": LANE_VERTICES,
            "steps_per_episode": EPISODE, "disable_dones": True,
            "seeds": {"scenarios": STRESS_SEED, "actions": ACTION_SEED, "reset": RESET_SEED},
            "l2": "inputs larger than L2 (per-GPU static pack > 126 MB for C1..C4)",
            "parallelism": f"scenario-sharded x{world} ({p['scaling']} scaling)"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict | None:
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for l in self.lines:
            parts = [p.strip() for p in l.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n: int) -> int:
    """`--gpus N` outside torchrun: re-run this command as N ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


# ---------------------------------------------------------------- reference arm
def _ref_workload(p: dict, n_scen: int):
    """(ZSIM bytes, rows, agents per row) of a bounded reference sample: the
    first `n_scen` scenarios of the same stress set (for C2 the per-row
    scenarios of their controlled actors).  Generated by oracle/_ref's copy of
    the workload generator -- the product library is never mapped here."""
    from oracle import refpy
    z = refpy.stress(n_scen, p["agents"], p["road_points"], seed=STRESS_SEED, c2=p["controlled"])
    if p["controlled"]:
        return refpy.controlled_expand(z), n_scen * p["agents"], 1
    return z, n_scen, p["agents"]


def cpu_baseline(p: dict) -> dict | None:
    """Reference simulator (oracle/_ref) timed on this host's cores over a
    bounded sample of the same workload (rank 0, N=1 only)."""
    from oracle import refpy
    from oracle.hostio import OracleConfig, random_actions
    if not refpy.available():
        return None
    n_scen = min(16 if p["controlled"] else 1024, p["total"])
    zsim, rows, apr = _ref_workload(p, n_scen)
    A, S = random_actions(EPISODE, rows, seed=ACTION_SEED)
    threads = os.cpu_count() or 1
    secs = refpy.bench(zsim, rows, 92, OracleConfig(**SIM_CONFIG), threads, 0, EPISODE, A, S)
    # single-thread leg on a C0-sized sample (64 rows), SURVEY 8d
    z1, r1, _ = _ref_workload(p, 1 if p["controlled"] else min(64, n_scen))
    r1 = min(r1, 64)
    A1, S1 = random_actions(EPISODE, r1, seed=ACTION_SEED)
    secs1 = refpy.bench(z1, r1, 92, OracleConfig(**SIM_CONFIG), 1, 0, EPISODE, A1, S1)
    return {"value": rows * apr * EPISODE / secs, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{rows} rows ({n_scen} of the {p['total']} {p['name']} scenarios) x {EPISODE} steps "
                      f"(observe+step), {threads} per-thread Env shards, oracle/_ref (-O2 -ffp-contract=off)",
            "seconds": secs,
            "value_1thread": r1 * apr * EPISODE / secs1,
            "sample_1thread": f"{r1} rows x {EPISODE} steps on 1 thread ({secs1:.2f} s)"}


def run_reference(args) -> None:
    """The reference's own CPU step (oracle/_ref = proj/src/core compiled in
    place) on this host's cores, same workload / metric / config keys."""
    world, rank, _ = dist_setup()
    if world != args.gpus:
        raise SystemExit(f"bench: WORLD_SIZE={world} but --gpus {args.gpus}")
    if rank != 0:
        return
    from oracle import refpy
    from oracle.hostio import OracleConfig, random_actions
    p = plan(args.config, world, args.scenarios)
    if not refpy.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libzsim_ref.so not built"}))
        return
    # a bounded sample per step: the CPU needs ~90 us per 32-agent scenario-step
    n_scen = min(32 if p["controlled"] else 4096, p["total"])
    zsim, B, apr = _ref_workload(p, n_scen)
    A, S = random_actions(EPISODE, B, seed=ACTION_SEED)
    threads = os.cpu_count() or 1
    secs = refpy.bench(zsim, B, 92, OracleConfig(**SIM_CONFIG), threads, args.warmup, args.steps, A, S)
    value = B * apr * args.steps / secs
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True,
        "scaling": p["scaling"], "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic: stress generator (seed {STRESS_SEED}), random actions (splitmix64 seed {ACTION_SEED})",
        "config": config_block(p, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{B} rows (the first {n_scen} of the {p['total']} scenarios) per step, "
                                   f"{args.steps} observe+step iterations, {threads} per-thread Env shards"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------- our arm
def run_ours(args) -> None:
    import torch

    world, rank, local = dist_setup()
    if world != args.gpus:
        raise SystemExit(f"bench: WORLD_SIZE={world} but --gpus {args.gpus}")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2312_15122_b200 as z
    from paper_2312_15122_b200.shard import StatsComm, shard_rows

    p = plan(args.config, world, args.scenarios)
    A_, P, controlled, rpr = p["agents"], p["road_points"], p["controlled"], p["rows_per_scenario"]
    lo, hi = shard_rows(p["total"], world, rank)
    S_ = hi - lo
    t_setup = time.perf_counter()
    env = z.Env.from_stress(z.StressConfig(count=S_, agents=A_, road_points=P, first_index=lo,
                                           flags=z.STRESS_C2 if controlled else 0), STRESS_SEED,
                            config=z.SimConfig(**SIM_CONFIG), device=local, controlled=controlled)
    setup_s = time.perf_counter() - t_setup
    if args.launch_policy:
        env.set_launch_policy(args.launch_policy)
    B = env.info.batch
    assert B == S_ * rpr, (B, S_, rpr)
    accel_all, steer_all = z.random_actions(EPISODE, p["total"] * rpr, seed=ACTION_SEED)
    accel = np.ascontiguousarray(accel_all[:, lo * rpr:hi * rpr])
    steer = np.ascontiguousarray(steer_all[:, lo * rpr:hi * rpr])
    del accel_all, steer_all
    dA = torch.from_numpy(accel).cuda()
    dS = torch.from_numpy(steer).cuda()
    s0, s1 = env.device_state(), env.device_state()
    so, ob = env.device_stepout(), env.device_obs()
    stats = torch.zeros(8, dtype=torch.int64, device="cuda")
    comm = StatsComm(rank, world, local) if world > 1 else None
    stream = torch.cuda.current_stream()

    def launch(k: int, cur, nxt, strm):
        """Launch k of a run: reset at t == 0, then the fused step."""
        t = k % EPISODE
        if t == 0:
            env.reset_device(RESET_SEED, cur, strm)
        env.step_observe_device(cur, dA[t].data_ptr(), dS[t].data_ptr(), nxt, so, ob, strm)
        return nxt, cur

    cur, nxt = s0, s1
    for k in range(args.warmup):
        cur, nxt = launch(k, cur, nxt, stream)
    env.check_errors(stream)
    # reset kernel duration (subtracted from the timed region for the kernel average)
    r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r0.record(stream)
    for _ in range(10):
        env.reset_device(RESET_SEED, cur, stream)
    r1.record(stream)
    torch.cuda.synchronize()
    reset_ms = r0.elapsed_time(r1) / 10

    # Timed region: exactly K launches (reset at every t % 91 == 0) as one CUDA graph.
    resets = sum(1 for k in range(args.steps) if k % EPISODE == 0)
    graph = None
    if not args.no_graph:
        gstream = torch.cuda.Stream()
        gstream.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=gstream, capture_error_mode="relaxed"):
            g_cur, g_nxt = s0, s1
            for k in range(args.steps):
                g_cur, g_nxt = launch(k, g_cur, g_nxt, gstream)
        final_state = g_cur
        stream = torch.cuda.current_stream()  # CUDAGraph.replay() launches on the current stream
        graph.replay()  # warm replay (untimed)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)  # let the sampler start before the timed region
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gc.collect()
    gc.disable()  # a collector pause in the launch loop would idle the GPU inside the timed region
    start.record(stream)
    if graph is not None:
        graph.replay()
        cur = final_state
    else:
        cur, nxt = s0, s1
        for k in range(args.steps):
            cur, nxt = launch(k, cur, nxt, stream)
    end.record(stream)
    torch.cuda.synchronize()
    gc.enable()
    clk = clocks.stop()
    if dist:
        dist.barrier()
    elapsed_ms = start.elapsed_time(end)
    env.check_errors(stream)
    # the fused kernel's average duration inside the timed region
    kern_ms = (elapsed_ms - resets * reset_ms) / args.steps
    t_max = torch.tensor([elapsed_ms], dtype=torch.float64, device="cuda")
    env.episode_stats(cur, stats.data_ptr(), stream)
    if dist:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)  # timing plumbing (max over ranks)
    if comm:
        comm.allreduce_stats(stats, stream)  # the one data collective: int64 stats over NCCL
        torch.cuda.synchronize()
        comm.check()
    elapsed_ms = float(t_max.item())
    agents_per_row = 1 if controlled else A_  # C2 counts controlled rows
    total_rows = p["total"] * rpr
    agent_steps = total_rows * agents_per_row * args.steps
    value = agent_steps / (elapsed_ms / 1e3)

    # ---- e2e through the host-vector API (the drop-in overloads) ----
    e2e = None
    if not args.no_e2e:
        st_h, nx_h = env.new_state(pinned=True), env.new_state(pinned=True)
        so_h, ob_h = env.new_stepout(pinned=True), env.new_obs(pinned=True)
        env.init_state(RESET_SEED, out=st_h)
        # C2 / C4 move 1-4 GB of observations per step over PCIe: a few steps suffice
        ke = min(args.steps, 3 if (controlled or B > 16384) else EPISODE)
        for t in range(min(3, ke)):
            env.step_observe(st_h, accel[t], steer[t], nx_h, so_h, ob_h)
        env.init_state(RESET_SEED, out=st_h)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for t in range(ke):
            env.step_observe(st_h, accel[t], steer[t], nx_h, so_h, ob_h)
            st_h, nx_h = nx_h, st_h
        t1 = time.perf_counter()
        e_s = torch.tensor([t1 - t0], dtype=torch.float64, device="cuda")
        if dist:
            dist.all_reduce(e_s, op=dist.ReduceOp.MAX)
        sb, sob, obb = env.layout
        h2d = sb + 8 * B  # state + actions
        d2h = sb + sob + obb
        e2e = {"value": total_rows * agents_per_row * ke / float(e_s.item()), "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": ke,
               "path": "Env.step_observe host-vector API (zsim_step_observe_host: step + observe of the next "
                       "state, observation streamed back in row chunks), pinned buffers"}

    policy = None
    if rank == 0 and world == 1 and not args.no_policy and not controlled and args.config == "C1":
        policy = measure_policy(env, ob, B, A_)

    if comm:
        comm.close()
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    per_scen = controlled_row_step_bytes(A_, P) if controlled else scenario_step_bytes(A_, P)
    peak, peak_src = hbm_peak()
    achieved = per_scen * B / (kern_ms / 1e3) / 1e9
    traffic = None
    tp = ROOT / "profiles" / "ncu_traffic.json"
    if tp.exists():
        try:
            tj = json.loads(tp.read_text())
            if tj.get("config") == args.config:
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            pass
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
        "scaling": p["scaling"], "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic: stress generator (seed {STRESS_SEED}; rank r owns its contiguous slice of the global "
                f"scenario set), random actions (splitmix64 seed {ACTION_SEED})",
        "config": config_block(p, world),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, ("bytes_per_row_step" if controlled else "bytes_per_scenario_step"): per_scen,
                     "units_per_launch": B,
                     "kernel": ("k_step_observe (fused step + observe)" if env.info.step_observe_kernels == 1
                                else "k_step_observe step+agents, then road/route top-k (per step)"),
                     "kernel_ms": kern_ms, "peak_source": peak_src},
        "gpu_launches": args.steps * env.info.step_observe_kernels + resets,
        "scenario_steps_per_s": p["total"] * args.steps / (elapsed_ms / 1e3),
        "controlled_agent_steps_per_s": total_rows * args.steps / (elapsed_ms / 1e3),
        "timing": {"mode": "cuda-graph (exactly `steps` fused launches + a reset every 91)" if graph is not None
                   else "eager launches",
                   "kernel_ms_source": "timed region minus resets x reset_ms, / steps (rank 0)",
                   "reset_ms": reset_ms, "resets_in_region": resets, "setup_s": setup_s,
                   "static_pack_mb_per_gpu": env.info.static_bytes / 1e6},
        "episode_stats": stats.cpu().tolist(),
    }
    assert kern_ms <= line["ms_per_step"] + 1e-9 or world > 1, (kern_ms, line["ms_per_step"])
    if e2e:
        line["e2e"] = e2e
    if policy:
        line["policy"] = policy
    if clk:
        line["clocks"] = clk
    if world == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline(p)
        if cb:
            line["cpu_baseline"] = cb
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def measure_policy(env, ob, B, A_):
    """NNPolicy::act on the device over the batch's
    observations, and the closed simulate -> act loop (zsim_rollout_policy,
    91 steps, one CUDA graph) -- reported beside the headline metric, for the
    default fp32 arithmetic (the reference's Model<float>) and the opt-in tf32
    tensor-core projections."""
    import torch

    import paper_2312_15122_b200 as z
    cfg = z.ModelConfig()
    params = z.init_params(cfg, 1)
    stream = torch.cuda.current_stream()
    rng = torch.arange(B, dtype=torch.int64, device="cuda")
    acc = torch.zeros(B, dtype=torch.int32, device="cuda")
    ste = torch.zeros_like(acc)
    lp = torch.zeros(B, dtype=torch.float32, device="cuda")
    val = torch.zeros_like(lp)
    peak_tf32 = None
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        peak_tf32 = float(json.loads(p.read_text())["bf16_tflops"]) / 2  # tf32 dense rate is half of bf16
    # tensor-core work per row: 10 token-tile projections (17 tokens x 128 x 128)
    # + the trunks (4 x 2 MLP matrices, value.in 160 -> 128), 2 flops per MAC
    tc_flops = (10 * 17 + 8) * 128 * 128 * 2 + 160 * 128 * 2
    out = {"rows": B}
    for prec in ("fp32", "tf32"):
        pol = z.NNPolicy(cfg, params, use_argmax=False, precision=prec)

        def act():
            pol.act_device(ob, B, rng.data_ptr(), acc.data_ptr(), ste.data_ptr(), lp.data_ptr(), val.data_ptr(),
                           stream=stream)
        for _ in range(3):
            act()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 20
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(n):
            act()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        env.rollout_policy_device(pol, 42, EPISODE, stream=stream)  # warm-up (allocates the scratch)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        gs = torch.cuda.Stream()
        with torch.cuda.stream(gs):
            with torch.cuda.graph(graph, stream=gs):
                env.rollout_policy_device(pol, 42, EPISODE, stream=gs)
        graph.replay()
        torch.cuda.synchronize()
        s2 = torch.cuda.current_stream()
        e0.record(s2)
        graph.replay()
        e1.record(s2)
        torch.cuda.synchronize()
        loop_ms = e0.elapsed_time(e1)
        achieved = tc_flops * B / (ms / 1e3) / 1e12
        out[prec] = {
            "precision": ("fp32 CUDA cores: the reference's Model<float> arithmetic (default)" if prec == "fp32"
                          else "tf32 projections on tcgen05, fp32 elsewhere (opt-in; logits ~1e-4 from fp32)"),
            "ms_per_act": ms, "rows_per_s": B / (ms / 1e3),
            "closed_loop": {"path": "zsim_rollout_policy: observe -> NNPolicy::act -> step, 91 steps, sampling, "
                                    "replayed from a CUDA graph",
                            "ms": loop_ms, "agent_steps_per_s": B * A_ * EPISODE / (loop_ms / 1e3)},
            "matmul_tflops": achieved}
        if prec == "tf32":
            out[prec]["roofline"] = {"bound": "tensor", "achieved": achieved, "peak": peak_tf32, "unit": "TFLOP/s",
                                     "frac": achieved / peak_tf32 if peak_tf32 else None,
                                     "peak_source": "MEASURED_PEAKS.json bf16_tflops / 2 (tf32)",
                                     "note": "the folded cross attention and the LayerNorm / softmax work run on "
                                             "the FP32 pipe and dominate the kernel time"}
        pol.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5 * EPISODE)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="C1", choices=sorted(CONFIGS))
    ap.add_argument("--scenarios", type=int, default=0, help="override the global scenario count (diagnostic)")
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of one CUDA graph")
    ap.add_argument("--no-policy", action="store_true", help="skip the on-device policy measurement")
    ap.add_argument("--launch-policy", type=int, default=0, choices=(0, 1, 2),
                    help="kernel arrangement: 0 auto, 1 fused step+observe, 2 split observation (diagnostic)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.steps < 1 or args.gpus < 1:
        raise SystemExit("bench: --steps and --gpus must be >= 1")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(spawn_ranks(args.gpus))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

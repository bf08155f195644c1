#!/usr/bin/env python
"""Throughput benchmark of the batched simulator step (BASELINE.json metric).

One "step" = one fused step+observe launch over the whole scenario batch
(Env::step then Env::observe of the stepped state, simcore.cpp:590-609).
Episodes are 91 steps long (T_log = 92); the state is re-initialised (reset
kernel, included in the timed region) every 91 steps.  Throughput runs use
`disable_dones = true` like the reference bench (simcore.cpp:669).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C1] [--impl ours|reference]

N > 1 is launched by torchrun (one process per GPU, NCCL); each rank simulates
its own shard of scenarios (weak scaling), no data-path collective; the only
collective is the all-reduce of the int64 episode-stats vector.
Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
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

# BASELINE.json configs; per-GPU shapes.
CONFIGS = {
    "C0": dict(scenarios=64, agents=32, road_points=2048,
               workload="C0: 64 scenarios x 32 agents, 2k roadgraph points, 91-step rollouts (CPU reference case)"),
    "C1": dict(scenarios=4096, agents=32, road_points=2048,
               workload="C1: 1xB200, 4096 scenarios x 32 agents, 2k roadgraph points, top-k 16 agents / 128 "
                        "polyline pts"),
    "C3": dict(scenarios=8192, agents=64, road_points=4096,
               workload="C3 per-GPU shard: 8192 scenarios x 64 agents, 4k roadgraph points"),
    "C4": dict(scenarios=16384, agents=128, road_points=8192,
               workload="C4 per-GPU shard at 8 GPUs: 16384 scenarios x 128 agents, 8k roadgraph points"),
    "C2": dict(scenarios=4096, agents=128, road_points=8192, controlled=True,
               workload="C2 dense: 4096 scenarios x 128 agents all controlled (524,288 ego rows), 8k roadgraph "
                        "points; agent-steps = controlled rows x steps (SURVEY 8a row 20)"),
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
                                          "--format=csv,noheader,nounits", "-lms", "100"],
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


def _ref_workload(c: dict, n_scen: int, seed: int):
    """(ZSIM bytes, rows, agents per row) of a reference-arm sample: stress
    scenarios, or for C2 the per-row scenarios of their controlled actors."""
    import paper_2312_15122_b200 as z
    controlled = bool(c.get("controlled"))
    zsim = z.stress_scenarios(z.StressConfig(count=n_scen, agents=c["agents"], road_points=c["road_points"],
                                             flags=z.STRESS_C2 if controlled else 0), seed)
    if controlled:
        return z.controlled_expand(zsim), n_scen * c["agents"], 1
    return zsim, n_scen, c["agents"]


def cpu_baseline(cfg_name: str, seed: int) -> dict | None:
    """Reference simulator (oracle/_ref) timed on this host's cores over a
    bounded sample of the same workload (rank 0, N=1 only)."""
    try:
        from oracle import refpy
    except Exception:
        return None
    if not refpy.available():
        return None
    import paper_2312_15122_b200 as z
    c = CONFIGS[cfg_name]
    n_scen = min(16 if c.get("controlled") else 1024, c["scenarios"])
    zsim, rows, apr = _ref_workload(c, n_scen, seed)
    A, S = z.random_actions(EPISODE, rows, seed=123)
    threads = os.cpu_count() or 1
    secs = refpy.bench(zsim, rows, 92, z.SimConfig(disable_dones=True), threads, 0, EPISODE, A, S)
    # single-thread leg on a C0-sized sample (64 rows), SURVEY 8d
    z1, r1, _ = _ref_workload(c, 1 if c.get("controlled") else min(64, n_scen), seed)
    r1 = min(r1, 64)
    A1, S1 = z.random_actions(EPISODE, r1, seed=123)
    secs1 = refpy.bench(z1, r1, 92, z.SimConfig(disable_dones=True), 1, 0, EPISODE, A1, S1)
    return {"value": rows * apr * EPISODE / secs, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{rows} rows ({n_scen} of the {c['scenarios']} {cfg_name} scenarios) x {EPISODE} steps "
                      f"(observe+step), {threads} per-thread Env shards, oracle/_ref (-O2 -ffp-contract=off)",
            "seconds": secs,
            "value_1thread": r1 * apr * EPISODE / secs1,
            "sample_1thread": f"{r1} rows x {EPISODE} steps on 1 thread ({secs1:.2f} s)"}


def run_reference(args) -> None:
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    import paper_2312_15122_b200 as z
    from oracle import refpy
    c = CONFIGS[args.config]
    if not refpy.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libzsim_ref.so not built"}))
        return
    # C2 has 524,288 rows: the reference times a bounded sample of them
    n_scen = min(32, c["scenarios"]) if c.get("controlled") else c["scenarios"]
    zsim, B, apr = _ref_workload(c, n_scen, 7)
    A, S = z.random_actions(EPISODE, B, seed=123)
    threads = os.cpu_count() or 1
    secs = refpy.bench(zsim, B, 92, z.SimConfig(disable_dones=True), threads, args.warmup, args.steps, A, S)
    value = B * apr * args.steps / secs
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (stress generator seed 7)",
        "config": {"workload": c["workload"], "scenarios": n_scen, "rows": B, "agents": c["agents"],
                   "road_points": c["road_points"], "steps_per_episode": EPISODE, "disable_dones": True},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{B} rows ({n_scen} scenarios), {args.steps} observe+step iterations, "
                                   f"{threads} threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def run_ours(args) -> None:
    import torch

    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2312_15122_b200 as z

    from paper_2312_15122_b200.shard import allreduce_stats, shard_rows
    c = CONFIGS[args.config]
    A_, P = c["agents"], c["road_points"]
    controlled = bool(c.get("controlled"))
    rpr = A_ if controlled else 1  # rows per scenario
    # weak scaling: the global set holds world x scenarios; rank r owns one contiguous shard
    lo, hi = shard_rows(c["scenarios"] * world, world, rank)
    S_ = hi - lo
    zsim = z.stress_scenarios(z.StressConfig(count=S_, agents=A_, road_points=P, first_index=lo,
                                             flags=z.STRESS_C2 if controlled else 0), 7)
    env = z.Env(zsim, config=z.SimConfig(disable_dones=True), device=local, controlled=controlled)
    if args.launch_policy:
        env.set_launch_policy(args.launch_policy)
    del zsim
    B = env.info.batch
    assert B == S_ * rpr, (B, S_, rpr)
    accel_all, steer_all = z.random_actions(EPISODE, c["scenarios"] * world * rpr, seed=123)
    accel = np.ascontiguousarray(accel_all[:, lo * rpr:hi * rpr])
    steer = np.ascontiguousarray(steer_all[:, lo * rpr:hi * rpr])
    dA = torch.from_numpy(accel).cuda()
    dS = torch.from_numpy(steer).cuda()
    s0, s1 = env.device_state(), env.device_state()
    so, ob = env.device_stepout(), env.device_obs()
    stats = torch.zeros(8, dtype=torch.int64, device="cuda")
    stream = torch.cuda.current_stream()

    k_state = {"k": 0}

    def one_step(cur, nxt, events=None):
        k = k_state["k"]
        t = k % EPISODE
        if t == 0:
            env.reset_device(42, cur, stream)
        if events is not None:
            events[0].record(stream)
        env.step_observe_device(cur, dA[t].data_ptr(), dS[t].data_ptr(), nxt, so, ob, stream)
        if events is not None:
            events[1].record(stream)
        k_state["k"] = k + 1
        return nxt, cur

    cur, nxt = s0, s1
    for _ in range(args.warmup):
        cur, nxt = one_step(cur, nxt)
    env.check_errors(stream)

    # Kernel timing (roofline): one eager episode, CUDA events around every fused launch.
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(EPISODE)]
    k_state["k"] = 0
    for i in range(EPISODE):
        cur, nxt = one_step(cur, nxt, kev[i])
    torch.cuda.synchronize()
    kern_ms_eager = float(np.mean([a.elapsed_time(b) for a, b in kev]))
    # reset kernel duration (subtracted from the graph-timed rollouts below)
    r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r0.record(stream)
    for _ in range(5):
        env.reset_device(42, cur, stream)
    r1.record(stream)
    torch.cuda.synchronize()
    reset_ms = r0.elapsed_time(r1) / 5

    # Timed region: whole rollouts (reset + 91 fused steps) replayed from a CUDA graph
    # (SURVEY 8d); a step count that is not a whole number of rollouts runs eagerly.
    use_graph = args.steps % EPISODE == 0 and not args.no_graph
    graph = None
    if use_graph:
        gstream = torch.cuda.Stream()
        gstream.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=gstream, capture_error_mode="relaxed"):
            g_cur, g_nxt = s0, s1
            env.reset_device(42, g_cur, gstream)
            for t in range(EPISODE):
                env.step_observe_device(g_cur, dA[t].data_ptr(), dS[t].data_ptr(), g_nxt, so, ob, gstream)
                g_cur, g_nxt = g_nxt, g_cur
        final_state = g_cur
        stream = torch.cuda.current_stream()  # CUDAGraph.replay() launches on the current stream
        graph.replay()  # warm replay
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)  # let the sampler start before the timed region
    resets = 0
    rollout_ms = []
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gc.collect()
    gc.disable()  # a collector pause in the launch loop would idle the GPU inside the timed region
    if use_graph:
        n_roll = args.steps // EPISODE
        rev = [torch.cuda.Event(enable_timing=True) for _ in range(n_roll + 1)]
        start.record(stream)
        rev[0].record(stream)
        for i in range(n_roll):
            graph.replay()
            rev[i + 1].record(stream)
        end.record(stream)
        resets = n_roll
        cur = final_state
    else:
        k_state["k"] = 0
        start.record(stream)
        for i in range(args.steps):
            resets += 1 if k_state["k"] % EPISODE == 0 else 0
            cur, nxt = one_step(cur, nxt)
        end.record(stream)
    torch.cuda.synchronize()
    gc.enable()
    clk = clocks.stop()
    if use_graph:
        rollout_ms = [rev[i].elapsed_time(rev[i + 1]) for i in range(n_roll)]
    # the fused kernel's average duration inside the timed region: CUDA events
    # around each graph rollout, minus its reset launch, over its 91 launches
    # (the eager per-launch-event figure includes launch gaps)
    kern_ms = (float(np.mean(rollout_ms)) - reset_ms) / EPISODE if rollout_ms else kern_ms_eager
    if dist:
        dist.barrier()
    elapsed_ms = start.elapsed_time(end)
    env.check_errors(stream)
    t_max = torch.tensor([elapsed_ms], dtype=torch.float64, device="cuda")
    env.episode_stats(cur, stats.data_ptr(), stream)
    if dist:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    allreduce_stats(stats)  # the one data collective: int64 episode stats over NCCL
    elapsed_ms = float(t_max.item())
    agents_per_row = 1 if controlled else A_  # C2 counts controlled rows
    agent_steps = B * agents_per_row * args.steps * world
    value = agent_steps / (elapsed_ms / 1e3)

    # ---- e2e through the host-vector API (the drop-in overloads) ----
    e2e = None
    if not args.no_e2e:
        st_h, nx_h = env.new_state(pinned=True), env.new_state(pinned=True)
        so_h, ob_h = env.new_stepout(pinned=True), env.new_obs(pinned=True)
        env.init_state(42, out=st_h)
        ke = min(args.steps, 3 if controlled else EPISODE)  # C2 moves 4 GB of observations per step over PCIe
        for t in range(min(3, ke)):
            env.step(st_h, accel[t], steer[t], nx_h, so_h)
            env.observe(nx_h, ob_h)
        env.init_state(42, out=st_h)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for t in range(ke):
            env.step(st_h, accel[t], steer[t], nx_h, so_h)
            env.observe(nx_h, ob_h)
            st_h, nx_h = nx_h, st_h
        t1 = time.perf_counter()
        e_s = torch.tensor([t1 - t0], dtype=torch.float64, device="cuda")
        if dist:
            dist.all_reduce(e_s, op=dist.ReduceOp.MAX)
        sb, sob, obb = env.layout
        h2d = 2 * sb + 8 * B  # step uploads state + actions, observe uploads state
        d2h = sb + sob + obb
        e2e = {"value": B * agents_per_row * ke * world / float(e_s.item()), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "steps": ke,
               "path": "Env.step + Env.observe host-vector API (zsim_step_host / zsim_observe_host), pinned buffers"}

    policy = None
    if rank == 0 and not args.no_policy and not controlled:
        policy = measure_policy(env, ob, B, A_)

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
        "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: stress generator (seed 7; rank r owns global rows [r*B, (r+1)*B)), random actions "
                "(splitmix64 seed 123)",
        "config": {"workload": c["workload"], "scenarios_per_gpu": S_, "rows_per_gpu": B, "agents": A_,
                   "road_points": P, "controlled": controlled,
                   "route_points": 2 * LANES * LANE_VERTICES, "lanes": LANES, "lane_vertices": LANE_VERTICES,
                   "steps_per_episode": EPISODE, "disable_dones": True,
                   "l2": f"inputs larger than L2 (static pack {env.info.static_bytes / 1e6:.0f} MB per GPU)",
                   "parallelism": f"scenario-sharded x{world}"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, ("bytes_per_row_step" if controlled else "bytes_per_scenario_step"): per_scen,
                     "kernel": ("k_step_observe (fused step + observe)" if env.info.step_observe_kernels == 1
                                else "k_step_observe step+agents, then road/route top-k (per step)"),
                     "kernel_ms": kern_ms, "peak_source": peak_src},
        "gpu_launches": args.steps * env.info.step_observe_kernels + resets,
        "scenario_steps_per_s": S_ * args.steps * world / (elapsed_ms / 1e3),
        "controlled_agent_steps_per_s": B * args.steps * world / (elapsed_ms / 1e3),
        "timing": {"mode": "cuda-graph rollouts (reset + 91 fused steps)" if use_graph else "eager launches",
                   "rollout_ms_median": float(np.median(rollout_ms)) if rollout_ms else None,
                   "rollout_ms_best": float(np.min(rollout_ms)) if rollout_ms else None,
                   "kernel_ms_source": "CUDA events around each graph rollout minus the reset launch, / 91"
                                       if rollout_ms else "one eager episode, CUDA events around each fused launch",
                   "kernel_ms_eager_events": kern_ms_eager, "reset_ms": reset_ms},
        "episode_stats": stats.cpu().tolist(),
    }
    if e2e:
        line["e2e"] = e2e
    if policy:
        line["policy"] = policy
    if clk:
        line["clocks"] = clk
    if world == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline(args.config, 7)
        if cb:
            line["cpu_baseline"] = cb
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def measure_policy(env, ob, B, A_):
    """NNPolicy::act on the device (tcgen05 tf32 projections)
    over the batch's observations, and the closed simulate -> act loop
    (zsim_rollout_policy, 91 steps) -- reported beside the headline metric."""
    import torch

    import paper_2312_15122_b200 as z
    cfg = z.ModelConfig()
    pol = z.NNPolicy(cfg, z.init_params(cfg, 1), use_argmax=False, precision="tf32")
    stream = torch.cuda.current_stream()
    rng = torch.arange(B, dtype=torch.int64, device="cuda")
    acc = torch.zeros(B, dtype=torch.int32, device="cuda")
    ste = torch.zeros_like(acc)
    lp = torch.zeros(B, dtype=torch.float32, device="cuda")
    val = torch.zeros_like(lp)

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
    # the whole closed loop (reset, 91 x [policy encoder + heads, fused step]) as one CUDA graph
    graph = torch.cuda.CUDAGraph()
    gs = torch.cuda.Stream()
    with torch.cuda.stream(gs):
        with torch.cuda.graph(graph, stream=gs):
            env.rollout_policy_device(pol, 42, EPISODE, stream=gs)
    graph.replay()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0.record(stream)
    graph.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    loop_ms = e0.elapsed_time(e1)
    # tensor-core work per row: 10 token-tile projections (17 tokens x 128 x 128)
    # + the trunks (4 x 2 MLP matrices, value.in 160 -> 128), 2 flops per MAC
    tc_flops = (10 * 17 + 8) * 128 * 128 * 2 + 160 * 128 * 2
    peak_tf32 = None
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        peak_tf32 = float(json.loads(p.read_text())["bf16_tflops"]) / 2  # tf32 dense rate is half of bf16
    achieved = tc_flops * B / (ms / 1e3) / 1e12
    return {"precision": "tf32 projections on tcgen05, fp32 elsewhere", "rows": B, "ms_per_act": ms,
            "rows_per_s": B / (ms / 1e3),
            "closed_loop": {"path": "zsim_rollout_policy: observe -> NNPolicy::act -> step, 91 steps, sampling, "
                                    "replayed from a CUDA graph",
                            "ms": loop_ms, "agent_steps_per_s": B * A_ * EPISODE / (loop_ms / 1e3)},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak_tf32, "unit": "TFLOP/s",
                         "frac": achieved / peak_tf32 if peak_tf32 else None,
                         "peak_source": "MEASURED_PEAKS.json bf16_tflops / 2 (tf32)",
                         "note": "the folded cross attention and the LayerNorm / softmax work run on the FP32 "
                                 "pipe and dominate the kernel time; the fraction is of the tf32 tensor peak"}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5 * EPISODE)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="C1", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of CUDA-graph rollouts")
    ap.add_argument("--no-policy", action="store_true", help="skip the on-device policy measurement")
    ap.add_argument("--launch-policy", type=int, default=0, choices=(0, 1, 2),
                    help="kernel arrangement: 0 auto, 1 fused step+observe, 2 split observation (diagnostic)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

"""Exercise every device kernel at small shapes, for compute-sanitizer.

    compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} python tools/sanitize.py

Covers: k_reset, k_step_observe fused (14-warp and 4-warp CTAs), the split
arrangement (step+agents, then road/route top-k), step-only / observe-only,
more than 32 agents (pruning, chunked ordering), C2 controlled rows, the
recorded device rollout + k_episode_finalize / k_episode_metrics /
k_metrics_sum / k_episode_stats, cut_sequences (k_seq_*), and the policy
kernels (k_policy_tc, k_policy_heads, k_policy_fp32) plus the closed loop.
Diagnostic tool; prints "sanitize: ok" at the end.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2312_15122_b200 as z


def run_env(env, steps, policies=(0,)):
    B = env.batch_size()
    A, S = z.random_actions(steps, B, seed=5)
    dA, dS = torch.from_numpy(A).cuda(), torch.from_numpy(S).cuda()
    for pol in policies:
        env.set_launch_policy(pol)
        s0, s1, so, ob = env.device_state(), env.device_state(), env.device_stepout(), env.device_obs()
        env.reset_device(42, s0)
        for t in range(steps):
            env.step_observe_device(s0, dA[t].data_ptr(), dS[t].data_ptr(), s1, so, ob)
            s0, s1 = s1, s0
        env.step_device(s0, dA[0].data_ptr(), dS[0].data_ptr(), s1, so)
        env.observe_device(s1, ob)
        stats = torch.zeros(8, dtype=torch.int64, device="cuda")
        env.episode_stats(s1, stats.data_ptr())
        torch.cuda.synchronize()
        env.check_errors()
    # host-vector API
    st = env.init_state(42)
    for t in range(2):
        st, _ = env.step(st, A[t], S[t])
        env.observe(st)
    return dA, dS


def main():
    small = "--small" in sys.argv
    # ego mode, C1-like shape at 3 scenarios; dones on so rows finish at different steps
    zs1 = z.stress_scenarios(z.StressConfig(count=3, agents=12, road_points=400, lane_vertices=24), 7)
    env = z.Env(zs1, config=z.SimConfig(disable_dones=False))
    run_env(env, 6, policies=(0, 1, 2))
    # > 32 agents (bound pruning, chunked ordering, 4-warp CTAs when smem is short)
    zs2 = z.stress_scenarios(z.StressConfig(count=2, agents=40, road_points=300, lane_vertices=16), 3)
    run_env(z.Env(zs2, config=z.SimConfig(disable_dones=True)), 4, policies=(1, 2))
    # C2 controlled rows
    zs3 = z.stress_scenarios(z.StressConfig(count=1, agents=34, road_points=300, lane_vertices=16, flags=z.STRESS_C2), 5)
    run_env(z.Env(zs3, config=z.SimConfig(disable_dones=True), controlled=True), 3, policies=(1, 2))
    # recorded device rollout, metrics, cut_sequences
    T = 5
    B = env.batch_size()
    A, S = z.random_actions(T, B, seed=9)
    dA, dS = torch.from_numpy(A).cuda(), torch.from_numpy(S).cuda()
    ep = env.device_episode(T)
    obs = [env.device_obs() for _ in range(T + 1)]
    env.rollout_device(42, T, dA.data_ptr(), dS.data_ptr(), T, episode=ep, obs=obs)
    env.episode_metrics(ep)
    env.cut_sequences_device(ep, obs, 3)
    torch.cuda.synchronize()
    # policy kernels: tf32 tensor-core path and fp32 path, argmax and sampling, closed loop
    cfg = z.ModelConfig()
    params = z.init_params(cfg, 1)
    for prec in ("tf32", "fp32"):
        for argmax in (True, False):
            pol = z.NNPolicy(cfg, params, use_argmax=argmax, precision=prec)
            rng = torch.arange(B, dtype=torch.int64, device="cuda")
            acc = torch.zeros(B, dtype=torch.int32, device="cuda")
            ste = torch.zeros_like(acc)
            lp = torch.zeros(B, dtype=torch.float32, device="cuda")
            val = torch.zeros_like(lp)
            pol.act_device(obs[1], B, rng.data_ptr(), acc.data_ptr(), ste.data_ptr(), lp.data_ptr(), val.data_ptr())
            if not small:
                env.rollout_policy_device(pol, 42, 3)
            torch.cuda.synchronize()
    print("sanitize: ok")


if __name__ == "__main__":
    main()

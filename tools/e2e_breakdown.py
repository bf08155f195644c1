"""Host-vector API cost breakdown at C1: step_host, observe_host, and the raw
pinned D2H bandwidth of an observation-sized copy.  Diagnostic tool."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2312_15122_b200 as z


def main(B=4096):
    zsim = z.stress_scenarios(z.StressConfig(count=B), 7)
    env = z.Env(zsim, config=z.SimConfig(disable_dones=True))
    A, S = z.random_actions(91, B, seed=1)
    st, nx = env.new_state(pinned=True), env.new_state(pinned=True)
    so, ob = env.new_stepout(pinned=True), env.new_obs(pinned=True)
    env.init_state(42, out=st)
    for t in range(3):
        env.step(st, A[t], S[t], nx, so)
        env.observe(nx, ob)
    n = 40
    t0 = time.perf_counter()
    for t in range(n):
        env.step(st, A[t], S[t], nx, so)
    t1 = time.perf_counter()
    for t in range(n):
        env.observe(nx, ob)
    t2 = time.perf_counter()
    dev = torch.empty(env.layout[2], dtype=torch.uint8, device="cuda")
    host = torch.empty(env.layout[2], dtype=torch.uint8, pin_memory=True)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    for _ in range(n):
        host.copy_(dev, non_blocking=True)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print({"step_host_ms": (t1 - t0) / n * 1e3, "observe_host_ms": (t2 - t1) / n * 1e3,
           "d2h_obs_ms": (t4 - t3) / n * 1e3, "obs_bytes": env.layout[2],
           "d2h_GBps": env.layout[2] / ((t4 - t3) / n) / 1e9})


if __name__ == "__main__":
    main()

"""The reference's step benchmark (sim::bench_step, simcore.cpp:654-699: step
only, zero actions, dones off, batch sizes 1..N) on the device and, for
continuity, the reference's own bench_step (oracle/_ref, one host thread) on
the same scenarios.  Prints bench_csv's columns for both.

    python tools/bench_step.py [scenarios] [steps]     (diagnostic tool)
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2312_15122_b200 as z

BATCH = [1, 16, 32, 64, 256, 1024, 4096]


def device_rows(zsim, n_scen, steps, warmup=10):
    lines = ["batch_size,mean_step_ms,amortized_us_per_scenario"]
    for bs in BATCH:
        idx = np.arange(bs) % n_scen  # ds indices i % ds.size(), as bench_step
        env = z.Env(zsim, indices=idx, config=z.SimConfig(disable_dones=True))
        a = torch.full((bs,), env.zero_accel_idx, dtype=torch.int32, device="cuda")
        s = torch.full((bs,), env.zero_steer_idx, dtype=torch.int32, device="cuda")
        s0, s1, so = env.device_state(), env.device_state(), env.device_stepout()
        env.reset_device(42, s0)
        for _ in range(warmup):
            env.step_device(s0, a.data_ptr(), s.data_ptr(), s1, so)
            s0, s1 = s1, s0
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            env.step_device(s0, a.data_ptr(), s.data_ptr(), s1, so)
            s0, s1 = s1, s0
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        lines.append(f"{bs},{ms:.6g},{ms * 1000.0 / bs:.6g}")
    return "\n".join(lines) + "\n"


def main():
    n_scen = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    zsim = z.stress_scenarios(z.StressConfig(count=n_scen), 7)  # C1 shapes: 32 agents, 2048 points
    print("# device (sm_100a step kernel, CUDA events), C1-shaped stress scenarios")
    print(device_rows(zsim, n_scen, steps), end="")
    from oracle import refpy
    if refpy.available():
        print("# reference sim::bench_step (oracle/_ref, 1 host thread), same scenarios")
        print(refpy.bench_step(zsim, BATCH, max(3, steps // 10), 2), end="")


if __name__ == "__main__":
    main()

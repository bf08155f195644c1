"""Time the step-only, observe-only and fused kernels on the C1 batch (device
events on the launching stream).  Diagnostic tool, not the bench."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2312_15122_b200 as z


def main(B=4096, A=32, P=2048, steps=40):
    zsim = z.stress_scenarios(z.StressConfig(count=B, agents=A, road_points=P), 7)
    env = z.Env(zsim, config=z.SimConfig(disable_dones=True))
    acc, st = z.random_actions(91, B, seed=123)
    dA, dS = torch.from_numpy(acc).cuda(), torch.from_numpy(st).cuda()
    s0, s1, so, ob = env.device_state(), env.device_state(), env.device_stepout(), env.device_obs()
    stream = torch.cuda.current_stream()
    res = {}
    for mode in ("step", "observe", "fused", "step+observe"):
        env.reset_device(42, s0, stream)
        for t in range(5):
            env.step_observe_device(s0, dA[t].data_ptr(), dS[t].data_ptr(), s1, so, ob, stream)
            s0, s1 = s1, s0
        torch.cuda.synchronize()
        ts = []
        for t in range(5, 5 + steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            if mode == "step":
                env.step_device(s0, dA[t].data_ptr(), dS[t].data_ptr(), s1, so, stream)
            elif mode == "observe":
                env.observe_device(s0, ob, stream)
            elif mode == "fused":
                env.step_observe_device(s0, dA[t].data_ptr(), dS[t].data_ptr(), s1, so, ob, stream)
            else:
                env.step_device(s0, dA[t].data_ptr(), dS[t].data_ptr(), s1, so, stream)
                env.observe_device(s1, ob, stream)
            e1.record(stream)
            ts.append((e0, e1))
            if mode != "observe":
                s0, s1 = s1, s0
        torch.cuda.synchronize()
        res[mode] = float(np.median([a.elapsed_time(b) for a, b in ts]))
    print({k: round(v * 1000, 1) for k, v in res.items()}, "us")


if __name__ == "__main__":
    main(*[int(x) for x in sys.argv[1:]])

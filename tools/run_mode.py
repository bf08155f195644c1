"""Run one kernel mode repeatedly on the C1 batch (for ncu captures)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2312_15122_b200 as z

mode = sys.argv[1] if len(sys.argv) > 1 else "fused"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
zsim = z.stress_scenarios(z.StressConfig(count=B), 7)
env = z.Env(zsim, config=z.SimConfig(disable_dones=True))
acc, st = z.random_actions(91, B, seed=123)
dA, dS = torch.from_numpy(acc).cuda(), torch.from_numpy(st).cuda()
s0, s1, so, ob = env.device_state(), env.device_state(), env.device_stepout(), env.device_obs()
env.reset_device(42, s0)
for t in range(8):
    if mode == "step":
        env.step_device(s0, dA[t].data_ptr(), dS[t].data_ptr(), s1, so)
    elif mode == "observe":
        env.observe_device(s0, ob)
        env.step_device(s0, dA[t].data_ptr(), dS[t].data_ptr(), s1, so)
    else:
        env.step_observe_device(s0, dA[t].data_ptr(), dS[t].data_ptr(), s1, so, ob)
    s0, s1 = s1, s0
torch.cuda.synchronize()
print("ok")

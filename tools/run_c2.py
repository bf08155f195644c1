"""Run a few C2 (all agents controlled) steps on a reduced batch (for ncu captures).
usage: python tools/run_c2.py [scenarios] [launch policy]   (diagnostic tool)"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2312_15122_b200 as z

S = int(sys.argv[1]) if len(sys.argv) > 1 else 512
zsim = z.stress_scenarios(z.StressConfig(count=S, agents=128, road_points=8192, flags=z.STRESS_C2), 7)
env = z.Env(zsim, config=z.SimConfig(disable_dones=True), controlled=True)
if len(sys.argv) > 2:
    env.set_launch_policy(int(sys.argv[2]))  # 1 fused, 2 split (the 524,288-row benchmark's arrangement)
B = env.info.batch
acc, st = z.random_actions(91, B, seed=123)
dA, dS = torch.from_numpy(acc).cuda(), torch.from_numpy(st).cuda()
s0, s1, so, ob = env.device_state(), env.device_state(), env.device_stepout(), env.device_obs()
env.reset_device(42, s0)
for t in range(6):
    env.step_observe_device(s0, dA[t].data_ptr(), dS[t].data_ptr(), s1, so, ob)
    s0, s1 = s1, s0
torch.cuda.synchronize()
print("ok", B)

"""Host staging + upload time of an Env (decode, route frames, pack, upload)
and the BatchStream overlap: wall time of iterating `n` batches with a
91-step device rollout each, with and without prefetch.  Diagnostic tool."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2312_15122_b200 as z


def main(B=4096, nb=4):
    zsim = z.stress_scenarios(z.StressConfig(count=B * nb), 7)
    torch.zeros(1).cuda()
    t0 = time.perf_counter()
    env = z.Env(zsim, indices=list(range(B)), config=z.SimConfig(disable_dones=True))
    torch.cuda.synchronize()
    t_env = time.perf_counter() - t0
    del env
    A, S = z.random_actions(91, B, seed=1)
    dA, dS = torch.from_numpy(A).cuda(), torch.from_numpy(S).cuda()
    res = {"B": B, "batches": nb, "env_create_s": t_env}
    for prefetch in (False, True):
        stream = z.BatchStream(zsim, B, config=z.SimConfig(disable_dones=True), prefetch=prefetch)
        t0 = time.perf_counter()
        sim = 0.0
        for env in stream:
            ep = env.device_episode(91)
            t1 = time.perf_counter()
            env.rollout_device(42, 91, dA.data_ptr(), dS.data_ptr(), 91, episode=ep)
            torch.cuda.synchronize()
            sim += time.perf_counter() - t1
            ep.close()
        res[f"wall_s_prefetch{int(prefetch)}"] = time.perf_counter() - t0
        res[f"sim_s_prefetch{int(prefetch)}"] = sim
        stream.close()
    print(res)


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])

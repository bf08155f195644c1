"""Time NNPolicy::act on device (zsim_policy_act) over B observation rows.
usage: python tools/policy_bench.py [B] [iters]   (diagnostic tool)"""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2312_15122_b200 as z
from paper_2312_15122_b200._abi import ObsView
from tests.test_policy import random_obs

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
obs = random_obs(B, np.random.default_rng(0))
dev = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in obs.items()}
view = ObsView()
for k, t in dev.items():
    setattr(view, k, C.cast(C.c_void_p(t.data_ptr()), C.POINTER(C.c_float)))
pol = z.NNPolicy(z.ModelConfig(), z.init_params(z.ModelConfig(), 1), use_argmax=False,
                 precision=sys.argv[3] if len(sys.argv) > 3 else "fp32")
rng = torch.arange(B, dtype=torch.int64, device="cuda")
a = torch.zeros(B, dtype=torch.int32, device="cuda")
s = torch.zeros_like(a)
lp = torch.zeros(B, dtype=torch.float32, device="cuda")
v = torch.zeros_like(lp)
stream = torch.cuda.current_stream()
run = lambda: pol.act_device(view, B, rng.data_ptr(), a.data_ptr(), s.data_ptr(), lp.data_ptr(), v.data_ptr(),
                             stream=stream)
for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(iters):
    run()
e1.record(stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / iters
# dense-contraction flops per row: 10 token-tile projections (self Q/K/V/O, cross Q/O x3) of 17 x 128 x 128
gemm_flops = 10 * 17 * 128 * 128 * 2
print(json.dumps({"rows": B, "ms": ms, "rows_per_s": B / ms * 1e3,
                  "projection_tflops": gemm_flops * B / ms / 1e9}))

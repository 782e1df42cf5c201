"""Worst-case |err| / (1e-4 + 1e-5|b|) of the FFMA kernel against the fp64
oracle for K = 4608 (512 -> 512 3x3, 28x28 maps, batch 32: whole-K units, so
the TMEM fold runs) as a function of the fold interval (DCONV_FLUSH_EVERY
stages).  Two images are checked.  Tool only."""
import os
import subprocess
import sys

if len(sys.argv) == 1:
    for fe in ("", "2", "4", "8", "16", "100000"):
        env = dict(os.environ)
        if fe:
            env["DCONV_FLUSH_EVERY"] = fe
        out = subprocess.run([sys.executable, __file__, "run"], env=env, capture_output=True,
                             text=True).stdout.strip()
        print(f"flush_every={fe or 'default'}: {out}", flush=True)
    sys.exit(0)

import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, ".")
from oracle import pyoracle as po  # noqa: E402
from paper_1809_10170_b200 import nets  # noqa: E402

ci, co, h, n = 512, 512, 30, 32
x = po.uniform((n, ci, h, h), 31, 0)
k = po.uniform((ci, co, 3, 3), 31, 1)
l = nets.Layer("a", ci, co, h, h, 3, 3, 1)
a = nets.Act(n, ci, h, h)
a.buf.copy_(torch.from_numpy(np.stack([po.pack_feature_map(x[i], 8) for i in range(n)])))
y = nets.Act(n, co, l.h_o, l.w_o)
nets.conv(l, n, a, nets.pack_weights(torch.from_numpy(k).cuda(), False), y)
torch.cuda.synchronize()
got = y.buf.cpu().numpy()
worst = 0.0
for i in (0, n - 1):
    want = po.pack_feature_map(po.conv_oracle64(x[i], k, 1), 8)
    worst = max(worst, float((np.abs(got[i] - want) / (1e-4 + 1e-5 * np.abs(want))).max()))
print(f"max err/tol {worst:.3f}")

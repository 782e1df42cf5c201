import time, sys, torch, numpy as np
sys.path.insert(0, '.')
from oracle import gpu_oracle as go, pyoracle as po
from paper_1809_10170_b200 import nets
l = nets.Layer("c", 256, 256, 58, 58, 3, 3, 1)
n = 32
x = nets.Act(n, 256, 58, 58); nets._fill(x.buf, 1, 2)
wd = torch.empty((256, 256, 3, 3), device="cuda"); nets._fill(wd, 1, 3)
torch.cuda.synchronize()
for i in range(3):
    t = time.time(); y = go.conv64_act(x, l, wd); torch.cuda.synchronize(); dt = time.time() - t
    print("oracle64 gpu", dt, "s", n * l.flops / dt / 1e12, "TFLOP/s", float(y.abs().max()), float(y[0,0,0,0,0]))
xc = x.buf[0].cpu().numpy(); kc = po.pack_kernel(wd.cpu().numpy(), 8, 8)
want = po.conv_oracle64_blocked(xc, kc, 256, 256, 1, 0, 1)
print("row0 equal", np.array_equal(want[:, 0], y[0, :, 0].float().cpu().numpy()))

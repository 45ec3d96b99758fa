"""Does the tensor-core conv slow down on a 36-float pixel stride (the
update-CNN feedback rows) against a dense 32-channel input? Times the stage
conv on [8, 288, 480] inputs (the last step's feature extent)."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2411_16680_b200 as q
from paper_2411_16680_b200 import workloads as wl

case = wl.config1()
m = q.Model(case.cfg, device=0)
dev = torch.device("cuda", 0)
B, H, W = 8, 288, 480
w = torch.randn(32, 97, 3, 3, device=dev) * 0.05
b = torch.randn(32, device=dev) * 0.1
y = torch.empty(B, H, W, 32, device=dev)
for ps in (32, 36, 40, 64):
    x = torch.randn(B, H, W, ps, device=dev)
    for _ in range(3):
        m.stage_conv3x3_fused(x, w, b, y, 32, ci0=0, impl=2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        m.stage_conv3x3_fused(x, w, b, y, 32, ci0=0, impl=2)
    e1.record()
    torch.cuda.synchronize()
    print(f"pixel stride {ps}: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us per conv (incl. weight prep)")
m.close()

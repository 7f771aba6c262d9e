import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, time, paper_2602_03002_b200 as md
d = torch.rand(4096, 2, 48, 64, device="cuda") * 9 + 0.5
cfg = md.SensorConfig()
out = torch.empty_like(d)
for i in range(3): md.apply_noise_dropout(d, cfg, d_max=[10.0, 10.0], step=i)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(50): md.apply_noise_dropout(d, cfg, d_max=[10.0, 10.0], step=i)
e1.record(); torch.cuda.synchronize()
print("noise kernel ms", e0.elapsed_time(e1) / 50)

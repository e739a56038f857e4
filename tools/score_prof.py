import sys
sys.path.insert(0, ".")
import torch, synth
from paper_2201_10369_b200 import api, points as PP
x, w = synth.layer_inputs(32, 256, 56, 56, 256, 3, "normal", "he", seed=0)
y, s, m = api.conv2d(torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), 1, 6, PP.family_n8_cd(2.0, 1.003), score=True)
torch.cuda.synchronize()
print(s.cpu().numpy())

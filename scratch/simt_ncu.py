import sys
sys.path.insert(0, '.')
import torch
from paper_1909_10616_b200 import tiletune as tt
n = int(sys.argv[1]); s = eval(sys.argv[2])
A = torch.randn(n, n, device='cuda'); B = torch.randn(n, n, device='cuda'); C = torch.empty(n, n, device='cuda')
for _ in range(5):
    tt.gemm(A, B, C, 1, s)
torch.cuda.synchronize()

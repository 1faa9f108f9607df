import torch
a = torch.rand(32768, 128, device='cuda', dtype=torch.float64).t()
b = torch.rand(32768, 32768, device='cuda', dtype=torch.float64)
for _ in range(3): c = a @ b
torch.cuda.synchronize()

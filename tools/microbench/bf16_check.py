import torch
a = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
b = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
c = a @ b
ref = a.float() @ b.float()
print("bf16 gemm max rel err", float((c.float() - ref).abs().max() / ref.abs().max()))

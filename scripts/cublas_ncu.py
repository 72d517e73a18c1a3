"""Library reference for the profile comparison (not the product path): one cuBLAS bf16 GEMM at 8192^3 (the
shape MEASURED_PEAKS.json's burst peak comes from) and at the config-2 gate/up shape (8192 x 11008 x 4096),
launched a few times so ncu can capture one of each. Measurement only."""
import torch

for (m, n, k) in ((8192, 8192, 8192), (8192, 11008, 4096)):
    a = torch.randn(m, k, device="cuda").bfloat16()
    b = torch.randn(k, n, device="cuda").bfloat16()
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()

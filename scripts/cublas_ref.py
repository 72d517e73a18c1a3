"""Library reference (not the product path): cuBLAS bf16 GEMM time on the dense shapes with the same FLOPs
as the grouped expert GEMMs of config 2, under the bench's protocol (L2 flushed, CUDA events), to show
how far the hand-written tcgen05 kernels are from the vendor library on this box."""
import json

import torch

dev = torch.device("cuda", 0)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)


def t(fn, n=20):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(n):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        out.append((a, b))
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in out) / n


res = {}
for name, (M, N, K) in {"gate_up_dense_equiv": (8192, 11008, 4096), "down_dense_equiv": (8192, 4096, 5504),
                        "square_8192": (8192, 8192, 8192)}.items():
    A = torch.randn(M, K, device=dev, dtype=torch.bfloat16)
    B = torch.randn(N, K, device=dev, dtype=torch.bfloat16)
    ms = t(lambda: torch.matmul(A, B.t()))
    res[name] = {"M": M, "N": N, "K": K, "ms": ms, "tflops": 2.0 * M * N * K / (ms * 1e-3) / 1e12}
# the grouped form cuBLAS would need: 8 per-expert GEMMs of 1024 rows
A = torch.randn(8, 1024, 4096, device=dev, dtype=torch.bfloat16)
B = torch.randn(8, 11008, 4096, device=dev, dtype=torch.bfloat16)
ms = t(lambda: torch.bmm(A, B.transpose(1, 2)))
res["gate_up_bmm_8x1024"] = {"ms": ms, "tflops": 2.0 * 8 * 1024 * 11008 * 4096 / (ms * 1e-3) / 1e12}
print(json.dumps(res))

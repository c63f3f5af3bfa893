"""One tcgen05 NS GEMM launch (for ncu): C = A B^T, bf16, M x N x K from argv."""
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2602_22437_b200 as R  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    R.ns_gemm_bf16(a, b, c)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    R.ns_gemm_bf16(a, b, c)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"{M}x{N}x{K}: {ms:.4f} ms, {2 * M * N * K / ms / 1e9:.1f} TFLOP/s")

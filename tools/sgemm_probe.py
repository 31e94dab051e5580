"""cuBLAS SGEMM (TF32 off) probe for ncu: what a library FFMA GEMM achieves here."""
import torch
torch.backends.cuda.matmul.allow_tf32 = False
a = torch.randn(8192, 8192, device="cuda")
b = torch.randn(8192, 8192, device="cuda")
for _ in range(3):
    c = a @ b
torch.cuda.synchronize()

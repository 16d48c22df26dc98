"""One standalone small-batch W4 GEMV launch per shape (ncu capture target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_02599_b200 import kernels
dev = torch.device("cuda")
for shape in os.environ.get("SHAPES", "28672x4096,6144x4096").split(","):
    n_out, k = map(int, shape.split("x"))
    for B in [int(b) for b in os.environ.get("PROBE_B", "1").split(",")]:
        w = (torch.randn(n_out, k, device=dev) * 0.02).to(torch.bfloat16)
        packed, scales = kernels.quantize_w4(w)
        x = torch.randn(16, k, device=dev).to(torch.bfloat16)
        for _ in range(2):
            kernels.gemm_w4(packed, scales, n_out, k, x, B, gemv=True)
        torch.cuda.synchronize()

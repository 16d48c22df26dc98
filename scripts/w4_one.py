"""One standalone QSUN W4 GEMM launch per shape (ncu capture target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_02599_b200 import kernels
dev = torch.device("cuda")
n_out, k = int(os.environ.get("N_OUT", 28672)), int(os.environ.get("K", 4096))
for B in [int(b) for b in os.environ.get("PROBE_B", "16,128").split(",")]:
    w = (torch.randn(n_out, k, device=dev) * 0.02).to(torch.bfloat16)
    packed, scales = kernels.quantize_w4(w)
    x = torch.randn(max(B, 16), k, device=dev).to(torch.bfloat16)
    for _ in range(2):
        kernels.gemm_w4(packed, scales, n_out, k, x, B)
    torch.cuda.synchronize()

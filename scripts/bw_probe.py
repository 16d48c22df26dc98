"""Reference points on this B200: read / copy bandwidth and cuBLAS bf16 GEMMs at decode shapes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_02599_b200 import kernels
dev = torch.device("cuda")
def t(fn, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it
x = torch.empty(2 * 1024**3, dtype=torch.bfloat16, device=dev).normal_()
y = torch.empty_like(x)
ms = t(lambda: x.sum(dtype=torch.float32)); print(f"read (torch.sum) {x.numel()*2/ms/1e6:.0f} GB/s")
ms = t(lambda: y.copy_(x)); print(f"copy {2*x.numel()*2/ms/1e6:.0f} GB/s")
del x, y
for n, k in [(6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336), (128256, 4096)]:
    W = (torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16)
    X = torch.randn(64, k, device=dev).to(torch.bfloat16)
    ms = t(lambda: X @ W.t())
    ws = kernels.gemm_workspace(n, k, 64, dev)
    out = torch.zeros(64, n, device=dev)
    Wb = kernels.block_weights(W)
    ms2 = t(lambda: kernels.gemm_bf16(Wb, X, 64, out=out, workspace=ws, shape=(n, k)))
    print(f"{n}x{k}: cuBLAS {ms*1e3:.1f} us ({n*k*2/ms/1e6:.0f} GB/s)   sun {ms2*1e3:.1f} us ({n*k*2/ms2/1e6:.0f} GB/s)")

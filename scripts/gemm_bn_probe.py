"""GEMM W-streaming rate vs batch (X bytes per stage) — is per-SM ingest the cap?"""
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
for n, k in [(28672, 4096), (128256, 4096)]:
    W = (torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16)
    Wb = kernels.block_weights(W)
    for B in (1, 16, 32, 64, 128, 256):
        X = torch.randn(max(16, (B + 15) // 16 * 16), k, device=dev).to(torch.bfloat16)
        ws = kernels.gemm_workspace(n, k, B, dev)
        out = torch.zeros(B, n, device=dev)
        ms = t(lambda: kernels.gemm_bf16(Wb, X, B, out=out, workspace=ws, shape=(n, k)))
        msc = t(lambda: X[:B] @ W.t())
        print(f"{n}x{k} B={B:3d}: sun {ms*1e3:6.1f} us {n*k*2/ms/1e6:5.0f} GB/s | cuBLAS {msc*1e3:6.1f} us {n*k*2/msc/1e6:5.0f} GB/s")

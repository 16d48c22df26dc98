"""Standalone QSUN W4 GEMM timing over batch sizes (CUDA events, L2 flushed between reps)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_02599_b200 import kernels

dev = torch.device("cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for n_out, k in [(28672, 4096), (4096, 14336), (6144, 4096), (4096, 4096)]:
    w = (torch.randn(n_out, k, device=dev) * 0.02).to(torch.bfloat16)
    packed, scales = kernels.quantize_w4(w)
    for B in (16, 64, 128, 256):
        x = torch.randn(B, k, device=dev).to(torch.bfloat16)
        ws = kernels.gemm_workspace(n_out, k, B, dev)
        out = torch.empty(B, n_out, device=dev)
        ts = []
        for it in range(6):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            kernels.gemm_w4(packed, scales, n_out, k, x, B, out=out, workspace=ws)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = sorted(ts[1:])[len(ts[1:]) // 2]
        wb = n_out * k // 2 + n_out * (k // 128) * 2
        print(f"W4 {n_out}x{k} B={B}: {t*1e3:.1f} us  {wb/t/1e6:.0f} GB/s (weights)", flush=True)

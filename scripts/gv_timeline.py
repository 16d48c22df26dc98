"""Per-CTA phase stamps of the small-batch W4 GEMV (sun_gemv_w4_stamped; slots 0 start,
1 setup done, 2 first stage landed, 3 last stage consumed, 5 last epilogue done, 6 exit)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_02599_b200 import _lib, kernels
lib = _lib.load()
dev = torch.device("cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
stream = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
tag0 = os.environ.get("TAG", os.environ.get("SUN_LIB", "")[-12:])
for n_out, k in [(28672, 4096), (4096, 14336), (6144, 4096), (4096, 4096)]:
    w = (torch.randn(n_out, k, device=dev) * 0.02).to(torch.bfloat16)
    packed, scales = kernels.quantize_w4(w)
    for B in (1, 16):
        x = torch.randn(16, k, device=dev).to(torch.bfloat16)
        out = torch.zeros(B, n_out, device=dev)
        ws = kernels.gemm_workspace(n_out, k, B, dev)
        st = torch.zeros(1024 * 16, dtype=torch.int64, device=dev)
        for it in range(3):
            st.zero_()
            flush.zero_()
            _lib.check(lib.sun_gemv_w4_stamped(packed.data_ptr(), scales.data_ptr(), n_out, k, x.data_ptr(), k, 16, B,
                                               out.data_ptr(), n_out, ws.data_ptr(), ws.numel(), stream(),
                                               st.data_ptr()))
            torch.cuda.synchronize()
        s = st.view(1024, 16).cpu().double()
        s = s[s[:, 0] > 0]
        t0 = s[:, 0].min()
        rel = lambda i: (s[:, i] - t0) / 1e3  # noqa: E731
        med = lambda v: float(v.median())  # noqa: E731
        wb = n_out * k // 2 + n_out * k // 64
        span = float((s[:, 6].max() - t0) / 1e3)
        print(f"{tag0:12s} {n_out}x{k} B={B:2d}: span {span:5.1f} us ({wb / span / 1e3:5.0f} GB/s) | start max "
              f"{float(rel(0).max()):.2f} | setup {med(rel(1) - rel(0)):.2f} | first stage {med(rel(2) - rel(1)):.2f} "
              f"max {float((rel(2) - rel(1)).max()):.2f} | main med {med(rel(3) - rel(2)):.2f} max "
              f"{float((rel(3) - rel(2)).max()):.2f} min {float((rel(3) - rel(2)).min()):.2f} | last-stage->epi done med {med(rel(5) - rel(3)):.2f} max "
              f"{float((rel(5) - rel(3)).max()):.2f} | exit med {med(rel(6)):.2f} max {float(rel(6).max()):.2f}",
              flush=True)

"""Per-role wait/work cycles inside the QSUN W4 GEMM (sun_gemm_w4_stamped)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_02599_b200 import _lib, kernels
lib = _lib.load()
dev = torch.device("cuda")
for n_out, k, B in [(28672, 4096, 16), (28672, 4096, 128)]:
    w = (torch.randn(n_out, k, device=dev) * 0.02).to(torch.bfloat16)
    packed, scales = kernels.quantize_w4(w)
    x = torch.randn(B, k, device=dev).to(torch.bfloat16)
    out = torch.zeros(B, n_out, device=dev)
    ws = kernels.gemm_workspace(n_out, k, B, dev)
    st = torch.zeros(4096 * 16, dtype=torch.int64, device=dev)
    for it in range(3):
        st.zero_()
        _lib.check(lib.sun_gemm_w4_stamped(packed.data_ptr(), scales.data_ptr(), n_out, k, x.data_ptr(), k, B, B,
                                           out.data_ptr(), n_out, ws.data_ptr(), ws.numel(),
                                           torch.cuda.current_stream().cuda_stream, st.data_ptr()))
        torch.cuda.synchronize()
    s = st.view(4096, 16).cpu().double()
    s = s[s[:, 0] > 0]
    t0 = s[:, 0].min()
    span = (s[:, 6].max() - t0) / 1e3
    print(f"W4 {n_out}x{k} B={B}: {len(s)} CTAs, span {span:.1f} us")
    loop = (s[:, 3] - s[:, 2]) / 1e3
    print(f"   main loop (first stage -> last MMA issue) med {loop.median():.2f} max {loop.max():.2f} us; "
          f"start->first stage med {((s[:, 2] - s[:, 0]) / 1e3).median():.2f}; last MMA->exit med {((s[:, 6] - s[:, 3]) / 1e3).median():.2f}")
    two = torch.tensor([((i + 1) * 224 // 148 - i * 224 // 148) == 2 for i in range(len(s))]) if n_out == 28672 else torch.ones(len(s), dtype=torch.bool)
    s = s[two]
    for i, nm in [(9, "mma wait X"), (10, "mma wait A"), (11, "mma issue"), (12, "cvt wait W"), (13, "cvt convert"),
                  (14, "cvt wait A slot"), (15, "cvt tmem st")]:
        c = s[:, i] / 1965.0
        print(f"   {nm:16s} med {c.median():7.2f} max {c.max():7.2f} us")

for B in (16, 64, 128):
    w = (torch.randn(28672, 4096, device=dev) * 0.02).to(torch.bfloat16)
    x = torch.randn(B, 4096, device=dev).to(torch.bfloat16)
    wb = kernels.block_weights(w)
    out = torch.zeros(B, 28672, device=dev)
    ts = []
    for it in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); kernels.gemm_bf16(wb, x, B, out=out, shape=(28672, 4096)); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"bf16 28672x4096 B={B}: {min(ts)*1e3:.1f} us")

"""Per-CTA timeline of one GEMM launch (globaltimer stamps) + event timing."""
import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_02599_b200 import _lib, kernels
lib = _lib.load()
dev = torch.device("cuda")
B = int(os.environ.get("B", "64"))
for n_out, k in [(6144, 4096), (4096, 4096), (4096, 14336), (28672, 4096)]:
    w = kernels.block_weights((torch.randn(n_out, k, device=dev) * 0.02).to(torch.bfloat16))
    x = torch.randn(B, k, device=dev).to(torch.bfloat16)
    out = torch.zeros(B, n_out, device=dev)
    ws = kernels.gemm_workspace(n_out, k, B, dev)
    st = torch.zeros(4096 * 16, dtype=torch.int64, device=dev)
    for it in range(3):
        st.zero_()
        _lib.check(lib.sun_gemm_bf16_stamped(w.data_ptr(), n_out, k, x.data_ptr(), k, B, B, out.data_ptr(), n_out, 0,
                                              ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream, st.data_ptr()))
        torch.cuda.synchronize()
    s = st.view(4096, 16).cpu().double()
    s = s[s[:, 0] > 0]
    t0 = s[:, 0].min()
    rel = (s - t0) / 1e3
    print(f"GEMM {n_out}x{k} B={B}: {len(s)} CTAs, kernel span {rel[:, 6].max():.1f} us ({n_out*k*2/(rel[:,6].max()*1e3):.0f} GB/s)")
    names = ["start", "setup", "first_stage", "last_mma", "first_acc", "epi_done", "exit", "-", "partial_parked", "csync1", "reduced", "epi_chunk"]
    for i, nm in enumerate(names):
        col = rel[:, i] if i != 7 else None
        if col is None or (s[:, i] == 0).all():
            continue
        print(f"   {nm:12s} min {col.min():7.2f} med {col.median():7.2f} max {col.max():7.2f} us")
    if os.environ.get("SLOW"):
        order = rel[:, 6].argsort(descending=True)[:8]
        for i in order.tolist():
            print("   cta", i, " ".join(f"{x:6.2f}" for x in rel[i, :14].tolist()))

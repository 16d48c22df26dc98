"""Per-CTA timeline of one GEMM launch (globaltimer stamps) + event timing."""
import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_02599_b200 import _lib, kernels
lib = _lib.load()
dev = torch.device("cuda")
for n_out, k in [(6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336), (128256, 4096)]:
    B = 64
    w = kernels.block_weights((torch.randn(n_out, k, device=dev) * 0.02).to(torch.bfloat16))
    x = torch.randn(64, k, device=dev).to(torch.bfloat16)
    out = torch.zeros(B, n_out, device=dev)
    ws = kernels.gemm_workspace(n_out, k, B, dev)
    st = torch.zeros(148 * 8 + 128, dtype=torch.int64, device=dev)
    for it in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(lib.sun_gemm_bf16_stamped(w.data_ptr(), n_out, k, x.data_ptr(), k, 64, B, out.data_ptr(), n_out, 0,
                                              ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream, st.data_ptr()))
        e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    allst = st.cpu().double()
    s = allst[:148 * 8].view(148, 8)
    s = s[s[:, 0] > 0]
    t0 = s[:, 0].min()
    rel = (s - t0) / 1e3
    gb = n_out * k * 2 / (ms / 1e3) / 1e9
    print(f"GEMM {n_out}x{k} B={B}: event {ms*1e3:.1f} us  ({gb:.0f} GB/s)")
    names = ["start", "setup", "first_stage", "last_mma", "first_acc", "epi_done", "exit"]
    for i, nm in enumerate(names):
        col = rel[:, i]
        print(f"   {nm:12s} min {col.min():7.2f} med {col.median():7.2f} max {col.max():7.2f} us")

    if n_out > 148 * 128:
        full = allst[148 * 8:148 * 8 + 64]
        iss = allst[148 * 8 + 64:148 * 8 + 128]
        base = s[0, 0]
        print("   CTA0 stage full times (us):", " ".join(f"{(x - base) / 1e3:.2f}" for x in full[:40]))
        print("   CTA0 reissue times (us):   ", " ".join(f"{(x - base) / 1e3:.2f}" for x in iss[8:40]))

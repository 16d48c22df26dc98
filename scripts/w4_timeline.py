"""Per-CTA phase stamps of the standalone QSUN W4 GEMM vs the bf16 GEMM on the same
shapes (sun_gemm_w4_stamped / sun_gemm_bf16_stamped; slots: 0 start, 1 setup done,
2 first stage landed at the MMA warp, 3 last MMA issued, 4 first accumulator ready,
5 epilogue done, 6 exit)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_02599_b200 import _lib, kernels
lib = _lib.load()
dev = torch.device("cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
stream = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731


def report(tag, s, span_us):
    s = s[s[:, 0] > 0]
    t0 = s[:, 0].min()
    rel = lambda i: (s[:, i] - t0) / 1e3  # noqa: E731
    med = lambda x: float(x.median())  # noqa: E731
    print(f"{tag}: {len(s)} CTAs, event {span_us:.1f} us, stamp span {float((s[:, 6].max() - t0) / 1e3):.1f} | start "
          f"med {med(rel(0)):.2f} max {float(rel(0).max()):.2f} | setup {med(rel(1) - rel(0)):.2f} | first stage "
          f"{med(rel(2) - rel(1)):.2f} | main loop med {med(rel(3) - rel(2)):.2f} max {float((rel(3) - rel(2)).max()):.2f}"
          f" | last MMA->acc {med(rel(4) - rel(3)):.2f} | epi {med(rel(5) - rel(4)):.2f} | exit max "
          f"{float(rel(6).max()):.2f}", flush=True)
    if os.environ.get("ROLE_CLOCKS"):  # -DSUN_W4_ROLE_CLOCKS build: cycles per role (CTA median, us at 1.965 GHz)
        names = {9: "mma wait X", 10: "mma wait A", 11: "mma issue", 12: "cvt wait W", 13: "cvt convert",
                 14: "cvt wait A slot", 15: "cvt tmem st+arrive"}
        print("   " + " | ".join(f"{nm} {float(s[:, i].median()) / 1965.0:.2f}" for i, nm in names.items()), flush=True)


for n_out, k in [(28672, 4096), (4096, 14336), (6144, 4096), (4096, 4096)]:
    w = (torch.randn(n_out, k, device=dev) * 0.02).to(torch.bfloat16)
    packed, scales = kernels.quantize_w4(w)
    wb = kernels.block_weights(w)
    for B in (16, 128):
        x = torch.randn(max(B, 16), k, device=dev).to(torch.bfloat16)
        out = torch.zeros(B, n_out, device=dev)
        ws = kernels.gemm_workspace(n_out, k, B, dev)
        st = torch.zeros(4096 * 16, dtype=torch.int64, device=dev)
        for name in (("w4",) if os.environ.get("W4ONLY") else ("w4", "bf16")):
            for it in range(3):
                st.zero_()
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                if name == "w4":
                    _lib.check(lib.sun_gemm_w4_stamped(packed.data_ptr(), scales.data_ptr(), n_out, k, x.data_ptr(), k,
                                                       x.shape[0], B, out.data_ptr(), n_out, ws.data_ptr(), ws.numel(),
                                                       stream(), st.data_ptr()))
                else:
                    _lib.check(lib.sun_gemm_bf16_stamped(wb.data_ptr(), n_out, k, x.data_ptr(), k, x.shape[0], B,
                                                         out.data_ptr(), n_out, 0, ws.data_ptr(), ws.numel(), stream(),
                                                         st.data_ptr()))
                e1.record()
                torch.cuda.synchronize()
            report(f"{os.environ.get('SUN_LIB', '')[-12:]:12s} {name:4s} {n_out}x{k} B={B}", st.view(4096, 16).cpu().double(), e0.elapsed_time(e1) * 1e3)

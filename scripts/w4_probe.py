"""QSUN W4 GEMM bottleneck probe: standalone sun_gemm_w4 timings (CUDA events, L2
flushed) for the library named by SUN_LIB (A/B variants built by
scripts/build_variant.sh: -DSUN_W4_NO_CVT skips the dequant arithmetic,
-DSUN_W4_NO_MMA skips the MMAs; both timing-only). PROBE_GEMV=1 times the
small-batch GEMV kernel for B <= 16."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_02599_b200 import kernels

dev = torch.device("cuda")
GEMV = os.environ.get("PROBE_GEMV") == "1"  # small-batch W4 GEMV kernel for B <= 16
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
shapes = [(28672, 4096), (4096, 14336), (6144, 4096), (4096, 4096)]
res = {}
for n_out, k in shapes:
    w = (torch.randn(n_out, k, device=dev) * 0.02).to(torch.bfloat16)
    packed, scales = kernels.quantize_w4(w)
    for B in [int(b) for b in os.environ.get("PROBE_B", "1,16,64,128").split(",")]:
        x = torch.randn(max(B, 16), k, device=dev).to(torch.bfloat16)
        ws = kernels.gemm_workspace(n_out, k, B, dev)
        out = torch.empty(B, n_out, device=dev)
        ts = []
        for it in range(8):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            kernels.gemm_w4(packed, scales, n_out, k, x, B, out=out, workspace=ws, gemv=GEMV and B <= 16)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = sorted(ts[2:])[len(ts[2:]) // 2]
        wb = n_out * k // 2 + n_out * (k // 128) * 2
        res[f"{n_out}x{k}/B{B}"] = round(t * 1e3, 1)
        print(f"{('gemv ' if GEMV and B <= 16 else '') + os.environ.get('SUN_LIB', 'default')[-30:]:30s} W4 {n_out}x{k} B={B}: {t*1e3:7.1f} us  {wb/t/1e6:6.0f} GB/s", flush=True)
print(json.dumps(res))

"""Token-parallel prefill throughput of one task module (8B-shaped, bf16)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_02599_b200.kvpool import KvPool, PageAllocator, pages_for
from paper_2603_02599_b200.modules import PrefillModule
from paper_2603_02599_b200.spec import SPECS
from paper_2603_02599_b200.weights import DeviceWeights, init_weights

spec = SPECS[os.environ.get("SPEC", "llama3.1-8b")]
dev = torch.device("cuda")
n, isl = 8, 1024
kv = KvPool(spec, n * pages_for(isl) + 4, dev)
alloc = PageAllocator(kv.num_pages)
pages = [alloc.alloc(pages_for(isl)) for _ in range(n)]
g = torch.Generator().manual_seed(0)
prompts = [torch.randint(0, spec.vocab, (isl,), generator=g).tolist() for _ in range(n)]
for mb, grouped in ((256, False), (64, True), (256, True)):
    pre = PrefillModule(spec, DeviceWeights(spec, init_weights(spec, 1, dev), dev, isl + 8), kv, mb, isl + 8, task_id=0,
                        grouped=grouped)
    pre.prefill(prompts[:1], pages[:1])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    first, _ = pre.prefill(prompts, pages)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{spec.name} max_batch={mb} grouped={grouped}: {n} x {isl} tokens in {dt * 1e3:.1f} ms = {n * isl / dt:.0f} prompt tok/s", flush=True)
    del pre

"""Diagnostic: one shared-decode step on the GPU vs the oracle, KV seeded from the oracle."""
import random, sys
sys.path.insert(0, '.')
import torch
from dataclasses import replace
import oracle.decoder_ref as R
from paper_2603_02599_b200.spec import TINY
from paper_2603_02599_b200.weights import init_weights, DeviceWeights
from paper_2603_02599_b200.kvpool import KvPool, PageAllocator, pages_for
from paper_2603_02599_b200.modules import SharedDecodeModule

cuda = torch.device('cuda')
def run(L, round_p, pdl=True):
    spec = replace(TINY, n_layers=L)
    w = init_weights(spec, 0)
    osp = R.OracleSpec(spec.vocab, spec.hidden, L, spec.n_q_heads, spec.n_kv_heads, spec.head_dim, spec.ffn, spec.rope_theta, spec.rms_eps)
    r = random.Random(1234)
    prompts = [[r.randrange(512) for _ in range(r.randint(16, 64))] for _ in range(8)]
    od = R.OracleDecoder(osp, w, 200)
    if round_p:
        orig = torch.softmax
        def sm(x, dim):
            m = x.max(dim=dim, keepdim=True).values
            p = torch.exp(x - m)
            return p.to(torch.bfloat16).float() / p.sum(dim=dim, keepdim=True)
        R.torch.softmax = sm
    caches, toks = [], []
    for p in prompts:
        lg, c = od.prefill(p); caches.append(c); toks.append(int(R.argmax_lowest(lg[None])[0]))
    kv = KvPool(spec, 8 * 8, cuda); kv.tensor.zero_()
    al = PageAllocator(kv.num_pages)
    pages = [al.alloc(pages_for(len(p) + 1)) for p in prompts]
    for i, p in enumerate(prompts):
        n = len(p)
        for l in range(L):
            K = caches[i]['k'][l]; V = caches[i]['v'][l]   # [n, nkv, d]
            for t in range(n):
                kv.tensor[pages[i][t // 16], l, 0, :, t % 16] = K[t].to(torch.bfloat16).to(cuda)
                kv.tensor[pages[i][t // 16], l, 1, :, t % 16] = V[t].to(torch.bfloat16).to(cuda)
    dec = SharedDecodeModule(spec, DeviceWeights(spec, w, cuda, 200), kv, 8, 200, use_pdl=pdl)
    bt = torch.zeros(8, dec.max_pages, dtype=torch.int32)
    for i, p in enumerate(pages): bt[i, :len(p)] = torch.tensor(p)
    nt = dec.decode(torch.tensor(toks, dtype=torch.int32), torch.tensor([len(p) for p in prompts], dtype=torch.int32), bt, graph=False).cpu()
    glog = dec.logits[:8].cpu()
    h = spec.hidden
    gres = dec.workspace[: 8 * h * 4].view(torch.float32).view(8, h).cpu()
    ores = []
    for i in range(8):
        pos = torch.tensor([len(prompts[i])])
        resid = od.w['embed'][torch.tensor([toks[i]])].clone()
        for l in range(L):
            resid = od._layer(l, resid, pos, caches[i]['k'], caches[i]['v'])
        ores.append(resid[0])
        # new-token KV written by the GPU QKV epilogue
        t = len(prompts[i]); pg = pages[i][t // 16]
        for l in range(L):
            gk = kv.tensor[pg, l, 0, :, t % 16].float().cpu(); ok = caches[i]['k'][l][-1]
            gv = kv.tensor[pg, l, 1, :, t % 16].float().cpu(); ov = caches[i]['v'][l][-1]
            if i == 0: print(f"  seq0 layer{l}: K maxdiff {(gk-ok).abs().max():.3g} (|k| {ok.abs().max():.3g}) V maxdiff {(gv-ov).abs().max():.3g}")
    ores = torch.stack(ores)
    print(f"  resid maxdiff {(gres-ores).abs().max():.3g} rel {((gres-ores).norm()/ores.norm()):.3g}")
    olog = torch.stack([(R.rmsnorm(ores[i:i+1], od.w['final_norm'], spec.rms_eps) @ od.w['lm_head'].t())[0] for i in range(8)])
    if round_p: R.torch.softmax = orig
    d = (glog - olog).abs()
    print(f"L={L} round_p={round_p}: max {d.max():.4g} mean {d.mean():.3g} logit std {olog.std():.3g} argmax eq {torch.equal(nt, R.argmax_lowest(olog).int())}")
run(1, False, False)
run(2, False, False)
run(4, False, False)

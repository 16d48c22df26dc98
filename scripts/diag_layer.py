"""Diagnostic: L=1 step, compare GPU workspace intermediates (q, attn, act, resid) with the oracle."""
import math, random, sys
sys.path.insert(0, '.')
import torch
from dataclasses import replace
import oracle.decoder_ref as R
from paper_2603_02599_b200.spec import TINY
from paper_2603_02599_b200.weights import init_weights, DeviceWeights
from paper_2603_02599_b200.kvpool import KvPool, PageAllocator, pages_for
from paper_2603_02599_b200.modules import SharedDecodeModule
cuda = torch.device('cuda')
spec = replace(TINY, n_layers=1)
L = 1
w = init_weights(spec, 0)
osp = R.OracleSpec(spec.vocab, spec.hidden, L, spec.n_q_heads, spec.n_kv_heads, spec.head_dim, spec.ffn, spec.rope_theta, spec.rms_eps)
r = random.Random(1234)
prompts = [[r.randrange(512) for _ in range(r.randint(16, 64))] for _ in range(8)]
od = R.OracleDecoder(osp, w, 200)
caches, toks = [], []
for p in prompts:
    lg, c = od.prefill(p); caches.append(c); toks.append(int(R.argmax_lowest(lg[None])[0]))
kv = KvPool(spec, 64, cuda); kv.tensor.zero_()
al = PageAllocator(kv.num_pages)
pages = [al.alloc(pages_for(len(p) + 1)) for p in prompts]
for i, p in enumerate(prompts):
    for t in range(len(p)):
        kv.tensor[pages[i][t // 16], 0, 0, :, t % 16] = caches[i]['k'][0][t].to(torch.bfloat16).to(cuda)
        kv.tensor[pages[i][t // 16], 0, 1, :, t % 16] = caches[i]['v'][0][t].to(torch.bfloat16).to(cuda)
dec = SharedDecodeModule(spec, DeviceWeights(spec, w, cuda, 200), kv, 8, 200, use_pdl=False)
bt = torch.zeros(8, dec.max_pages, dtype=torch.int32)
for i, p in enumerate(pages): bt[i, :len(p)] = torch.tensor(p)
pos = [len(p) for p in prompts]
dec.decode(torch.tensor(toks, dtype=torch.int32), torch.tensor(pos, dtype=torch.int32), bt, graph=False)
torch.cuda.synchronize()
ws = dec.workspace.cpu()
h, qd, f, B = 256, 512, 688, 8
def view(off, n, dt): return ws[off:off + n * (4 if dt == torch.float32 else 2)].view(dt)
g_resid = view(0, B*h, torch.float32).view(B, h).float()
g_q = view(16384, B*qd, torch.bfloat16).view(B, qd).float()
g_attn = view(24576, B*qd, torch.bfloat16).view(B, qd).float()
g_act = view(40960, B*f, torch.bfloat16).view(B, f).float()
W = od.w; d = 64; nq, nkv = 8, 2
for i in range(8):
    resid = W['embed'][toks[i]][None].clone()
    xn = R.rmsnorm(resid, W['l0.attn_norm'], spec.rms_eps)
    q = xn @ W['l0.wq'].t(); k = xn @ W['l0.wk'].t(); v = xn @ W['l0.wv'].t()
    cs, sn = od.cos[pos[i]][None, None], od.sin[pos[i]][None, None]
    q = R.bf(R.rope(q.view(1, nq, d), cs, sn)); k = R.bf(R.rope(k.view(1, nkv, d), cs, sn)); v = R.bf(v.view(1, nkv, d))
    K = torch.cat([caches[i]['k'][0], k]); V = torch.cat([caches[i]['v'][0], v])
    out = torch.empty(nq, d)
    for hh in range(nq):
        s = (K[:, hh // 4] @ q[0, hh]) / math.sqrt(d); out[hh] = torch.softmax(s, 0) @ V[:, hh // 4]
    attn = R.bf(out.reshape(1, -1))
    resid2 = resid + attn @ W['l0.wo'].t()
    xn2 = R.rmsnorm(resid2, W['l0.ffn_norm'], spec.rms_eps)
    g = xn2 @ W['l0.wg'].t(); u = xn2 @ W['l0.wu'].t()
    act = R.bf(g / (1 + torch.exp(-g)) * u)
    resid3 = resid2 + act @ W['l0.wd'].t()
    print("ctx", pos[i] + 1)
    def cmp(name, a, b):
        dd = (a - b).abs(); print(f"seq{i} {name}: maxdiff {dd.max():.3g} mismatches {(dd>0).float().mean():.3f} |ref| {b.abs().max():.3g}")
    cmp('q', g_q[i], q.reshape(-1)); cmp('attn', g_attn[i], attn[0]); cmp('act', g_act[i], act[0]); cmp('resid', g_resid[i], resid3[0])

"""Quick timing probe of the forward kernel (dev tool; bench.py is the contract)."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import hla_synth
import paper_2511_05832_b200 as hla

def t_ms(fn, iters=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters

for name, kind, g, w, B, H, d in [("cfg2", "HWA", 64, 16, 16, 8, 64), ("cfg2rm", "WSA", 64, 16, 16, 8, 64),
                                  ("cfg3", "HSA", 64, 16, 16, 8, 64), ("cfg3rm", "SA", 64, 16, 16, 8, 64),
                                  ("cfg4", "HNA", 128, 7, 16, 12, 64), ("cfg4rm", "NA2D", 128, 7, 16, 12, 64),
                                  ("dense2", "DENSE", 64, 1, 16, 8, 64)]:
    N = g * g
    q, k, v, do = hla_synth.attention_inputs(B, N, H, d, device="cuda")
    L = hla.HilbertLocalAttention(kind, g, g, w, w, B, H, d, device="cuda")
    ms = t_ms(lambda: hla.hla_attn_fwd(L.desc, L.mask, q, k, v, 0.0, L.o, L.lse))
    tiles = B * H * L.nnz
    flops = 4 * 128 * 128 * d * tiles
    byts = B * H * N * (8 * d + 4)
    print("%-7s fwd %.4f ms  tiles=%d  %.1f TF/s  %.0f GB/s(compulsory)" % (name, ms, tiles, flops / ms / 1e9, byts / ms / 1e6))
    if L.hilbert:
        ms = t_ms(lambda: hla.hla_hilbert_perm(g, g, 0, (q, k, v), (L.qs, L.ks, L.vs)))
        print("        perm(q,k,v) %.4f ms  %.0f GB/s" % (ms, 3 * 2 * q.numel() * 2 / ms / 1e6))

import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_05832_b200 import api
for d in (64, 32):
    src = torch.randn(4096, 8, d, device="cuda").bfloat16()
    idx = torch.randperm(4096, device="cuda")[:128].int().contiguous()
    for box_h in (1,):
        try:
            out = api.hla_debug_gather4(src, idx, 3, box_h)
            torch.cuda.synchronize()
            ref = src[idx.long(), 3]
            print("d", d, "box_h", box_h, "match", torch.equal(out, ref), "max err", (out.float() - ref.float()).abs().max().item())
        except Exception as e:
            print("d", d, "box_h", box_h, "ERROR", e)
            break

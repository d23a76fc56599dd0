import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_10652_b200 import kernels as K
for (M, N, Kd, act, bias, res) in [(4096, 4096, 1024, 0, False, False), (4096, 4096, 1024, 1, True, False),
                                   (2048 + 128 + 64, 1024, 4096, 0, True, True), (1000, 512, 256, 0, False, False)]:
    for pair in (1, 0):
        torch.manual_seed(3)
        a = torch.randn(M, Kd, device="cuda").bfloat16()
        w = (torch.randn(N, Kd, device="cuda") / Kd ** 0.5).bfloat16()
        bv = torch.randn(N, device="cuda").bfloat16() if bias else None
        rv = torch.randn(M, N, device="cuda").bfloat16() if res else None
        o = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        try:
            K.gemm(a, Kd, w, Kd, o, M, N, Kd, out_s=(0, 0, N, 1), bias=bv, act=act, res=rv, bn=256, cta_pair=pair)
            torch.cuda.synchronize()
            ref = a.float() @ w.float().T + (bv.float() if bias else 0)
            if act == 1:
                ref = torch.nn.functional.gelu(ref)
            if res:
                ref = ref + rv.float()
            print(M, N, Kd, act, bias, res, "pair", pair, "rel", ((o.float() - ref).abs().max() / ref.abs().max()).item(), flush=True)
        except Exception as e:
            print(M, N, Kd, act, bias, res, "pair", pair, "ERR", e, flush=True)

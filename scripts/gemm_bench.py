"""Microbenchmark of the tcgen05 GEMM (ac_kernel_gemm) on the GPT/AF linear shapes
vs torch.matmul (cuBLAS), CUDA events, L2 not flushed (operands re-read per launch)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_10652_b200 import kernels as K  # noqa: E402


def t_ms(fn, it=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it


def main():
    torch.manual_seed(0)
    only = sys.argv[1:]  # name bn act: one configuration, 2 launches (for ncu)
    shapes = [("ffn1", 16384, 4096, 1024, 1, True), ("ffn2", 16384, 1024, 4096, 0, False),
              ("proj", 16384, 1024, 1024, 0, False), ("qkv", 16384, 3072, 1024, 0, False),
              ("af_proj", 1 << 20, 128, 128, 0, False),
              # row chunks of the fused-attention block's FFN / output projection
              ("ffn1_c", 1024, 4096, 1024, 1, True), ("ffn2_c", 1024, 1024, 4096, 0, False),
              ("proj_c", 1024, 1024, 1024, 0, False), ("ffn1_c2", 2048, 4096, 1024, 1, True),
              ("ffn2_c2", 2048, 1024, 4096, 0, False)]
    for name, M, N, Kd, act, bias in shapes:
        if only and name != only[0]:
            continue
        a = torch.randn(M, Kd, device="cuda").bfloat16()
        w = (torch.randn(N, Kd, device="cuda") / Kd ** 0.5).bfloat16()
        bb = (torch.randn(N, device="cuda") * 0.02).bfloat16() if bias else None
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        fl = 2.0 * M * N * Kd
        if only:
            bn, aa = int(only[1]), int(only[2])
            for _ in range(2):
                K.gemm(a, Kd, w, Kd, out, M, N, Kd, out_s=(0, 0, N, 1), act=aa, bias=bb if aa else None, bn=bn)
            torch.cuda.synchronize()
            return
        tc = t_ms(lambda: torch.matmul(a, w.t()))
        res = [f"{name:8s} M={M} N={N} K={Kd}: cuBLAS {tc*1e3:7.1f} us {fl/tc/1e9:6.0f} TF/s"]
        for bn in ((0, 64, 128, 256) if M <= 4096 else (128, 256)):
            if bn > N:
                continue
            for aa in sorted({0, act}):
                f = lambda: K.gemm(a, Kd, w, Kd, out, M, N, Kd, out_s=(0, 0, N, 1), act=aa, bias=bb if aa else None, bn=bn)
                try:
                    t = t_ms(f)
                    res.append(f"   ours bn={bn} act={aa}: {t*1e3:7.1f} us {fl/t/1e9:6.0f} TF/s")
                except Exception as e:
                    res.append(f"   ours bn={bn} act={aa}: {e}")
        for pair in (0, 1):   # BN = 256 as single CTAs / CTA pairs (cta_group::2)
            f = lambda: K.gemm(a, Kd, w, Kd, out, M, N, Kd, out_s=(0, 0, N, 1), act=act, bias=bb if act else None,
                               bn=256, cta_pair=pair)
            try:
                t = t_ms(f)
                res.append(f"   ours bn=256 cta_pair={pair} act={act}: {t*1e3:7.1f} us {fl/t/1e9:6.0f} TF/s")
            except Exception as e:
                res.append(f"   ours bn=256 cta_pair={pair}: {e}")
        if act:
            ref = torch.nn.functional.gelu(torch.matmul(a.float(), w.float().t()) + bb.float())
            K.gemm(a, Kd, w, Kd, out, M, N, Kd, out_s=(0, 0, N, 1), act=act, bias=bb, bn=256)
            torch.cuda.synchronize()
            res.append(f"   gelu max abs err {(out.float() - ref).abs().max().item():.3e}")
        print("\n".join(res), flush=True)


if __name__ == "__main__":
    main()

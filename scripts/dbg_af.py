"""Which AF chunk plans are bitwise equal to the unchunked run (fused / unfused)."""
import os
import sys

import faulthandler

import torch

faulthandler.dump_traceback_later(40, exit=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import gpu_util as gu  # noqa: E402
from oracle import memory, workloads  # noqa: E402
from paper_2401_10652_b200 import api  # noqa: E402

NRES = int(sys.argv[1]) if len(sys.argv) > 1 else 64
PI = int(sys.argv[2]) if len(sys.argv) > 2 else -1
for nres in (NRES,):
    og = workloads.tri_attn_pair(nres, 128, 4, 32, "bf16", name="af_small")
    cg = gu.c_graph(og)
    p = api.ac_plan(cg, int(0.2 * memory.profile(og).peak_bytes))
    print(nres, "ac_plan:", p.serialize().replace("\n", " | "))
    vals, dev = gu.make_values(og, 0)
    for flag in ("0", "1"):
        os.environ["AC_FUSE_SOFTMAX"] = flag
        base, _ = gu.run(cg, gu.empty_plan(cg), og, dev)
        for txt in [p, "autochunk-plan 1\nregion s=row_scores e=row_pv n=4 dims=0\n",
                    "autochunk-plan 1\nregion s=row_scores e=row_pv n=4 dims=1\n",
                    "autochunk-plan 1\nregion s=col_scores e=col_pv n=4 dims=0\n",
                    "autochunk-plan 1\nregion s=col_scores e=col_pv n=4 dims=1\n"][PI:PI + 1 if PI >= 0 else None]:
            try:
                plan = api.plan_parse(cg, txt) if isinstance(txt, str) else txt
            except Exception as e:
                print("  parse fail", txt.replace("\n", " | "), e)
                continue
            got, ex = gu.run(cg, plan, og, dev)
            torch.cuda.synchronize()
            o = og.outputs[0]
            d = (got[o].float() - base[o].float()).abs()
            print(f"  nres={nres} fuse={flag} {plan.serialize().splitlines()[1:]} equal={torch.equal(got[o], base[o])} maxdiff={d.max().item():.3g} nbad={(d > 0).sum().item()}", flush=True)

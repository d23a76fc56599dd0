"""compute-sanitizer over small runs of every kernel path.  memcheck with the
PyTorch caching allocator off, so each tensor is its own allocation and any
read or write past a tensor's end is reported (e.g. aux loads of a ragged last
column tile); racecheck (shared-memory hazards between the warp roles) and
synccheck (barrier misuse) over the kernels with warp-specialised pipelines:
the f2 chain with the chunk-loop overlap (epochs, dynamic tiles), the paired
triangle chain, the fused attention, a vectorised-epilogue GEMM, and the
multi-rank executor on an in-process communicator.  GPU only."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
sys.path[:0] = [%(root)r, %(root)r + "/tests"]
import torch
import gpu_util as gu
from oracle import workloads
from paper_2401_10652_b200 import api, kernels as K

torch.manual_seed(0)
# ragged N (640 = 2.5 x 256-column tiles) with bias + residual: the row epilogue
M, N, Kd = 300, 640, 256
a = torch.randn(M, Kd, device="cuda").bfloat16()
w = torch.randn(N, Kd, device="cuda").bfloat16()
bias = torch.randn(N, device="cuda").bfloat16()
res = torch.randn(M, N, device="cuda").bfloat16()
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
K.gemm(a, Kd, w, Kd, out, M, N, Kd, out_s=(0, 0, N, 1), bias=bias, act=1, res=res)
torch.cuda.synchronize()
for og, txt in [
    (workloads.block("attn_only", 640, 640, 10, 0, False, "bf16", name="u"),
     "autochunk-plan 1\nregion s=scores e=pv n=3 dims=0\n"),
    (workloads.block("transformer", 1024 + 96, 256, 4, 1024, True, "bf16", name="g"),
     "autochunk-plan 1\nregion s=scores e=pv n=4 dims=0\n"),
    (workloads.block("transformer", 1024, 256, 4, 1024, True, "bf16", name="g2"),
     "autochunk-plan 1\nregion s=proj_q e=ffn2 n=4 dims=0\n"),
    (workloads.tri_attn_pair(48, 128, 4, 32, "bf16", name="af"),
     "autochunk-plan 1\nregion s=row_scores e=row_pv n=4 dims=0\n"),
    # short row chunks of the triangle chains: paired 64-row scores / PV (M = 40, ragged keys)
    (workloads.tri_attn_pair(80, 128, 4, 32, "bf16", name="af2"),
     "autochunk-plan 1\nregion s=row_scores e=row_pv n=2 dims=1\nregion s=col_scores e=col_pv n=3 dims=0\n"),
    # fused attention (NEXT f1), ragged rows / keys, causal chunks
    (workloads.block("transformer_fa", 200, 256, 4, 512, True, "bf16", name="fa"),
     "autochunk-plan 1\nregion s=attn e=ffn2 n=3 dims=0\n"),
    # 3-block stack with the chunk-loop overlap (PDL launches, epochs)
    (workloads.transformer(512, 256, 4, 512, True, "bf16", name="st", layers=2),
     "autochunk-plan 1\nregion s=L0_scores e=L0_pv n=4 dims=0\nregion s=L1_scores e=L1_pv n=2 dims=0\n"),
]:
    cg = gu.c_graph(og)
    vals, dev = gu.make_values(og, 0)
    for t in [txt, "autochunk-plan 1\n"]:
        gu.run(cg, api.plan_parse(cg, t), og, dev)
        torch.cuda.synchronize()
# forced PV split-K with the online fold (granule partials + (max, sum), counters in the
# control block under the overlap), and causal chains without the overlap
import os
for env in ({"AC_PV_SPLITK": "1"}, {"AC_OVERLAP_CAUSAL": "0"}):
    os.environ.update(env)
    for causal in (False, True):
        og = workloads.block("attn_only", 640 + 96, 256, 4, 0, causal, "bf16", name="sk")
        cg = gu.c_graph(og)
        vals, dev = gu.make_values(og, 1)
        for t in ["autochunk-plan 1\nregion s=scores e=pv n=3 dims=0\n", "autochunk-plan 1\n"]:
            gu.run(cg, api.plan_parse(cg, t), og, dev)
            torch.cuda.synchronize()
    for k in env:
        del os.environ[k]
print("SANITIZER-RUN-OK")
"""


SCRIPT_SYNC = r"""
import sys, threading
sys.path[:0] = [%(root)r, %(root)r + "/tests"]
import torch
import gpu_util as gu
from oracle import workloads
from paper_2401_10652_b200 import api

for og, txt in [
    (workloads.block("transformer", 512, 256, 4, 512, True, "bf16", name="g"),
     "autochunk-plan 1\nregion s=scores e=pv n=4 dims=0\n"),
    (workloads.block("attn_only", 384, 256, 4, 0, False, "bf16", name="u"),
     "autochunk-plan 1\nregion s=scores e=pv n=3 dims=0\n"),
    (workloads.tri_attn_pair(48, 128, 4, 32, "bf16", name="af"),
     "autochunk-plan 1\nregion s=row_scores e=row_pv n=2 dims=1\n"),
    (workloads.block("transformer_fa", 256, 256, 4, 512, True, "bf16", name="fa"),
     "autochunk-plan 1\nregion s=attn e=ffn2 n=2 dims=0\n"),
]:
    cg = gu.c_graph(og)
    vals, dev = gu.make_values(og, 0)
    gu.run(cg, api.plan_parse(cg, txt), og, dev)
    torch.cuda.synchronize()
# two in-process ranks (threads) through the multi-rank executor
og = workloads.block("transformer", 512, 256, 4, 512, True, "bf16", name="mr")
cg = gu.c_graph(og)
_, dev = gu.make_values(og, 0)
plan = api.plan_parse(cg, "autochunk-plan 1\nregion s=scores e=pv n=4 dims=0\n")
comms = api.Comm.local(2)
ins = {t: dev[t] for t in og.inputs + og.weights}
exs, outs = [], []
for r in range(2):
    ws = torch.empty(plan.workspace_bytes(r, 2), dtype=torch.uint8, device="cuda")
    exs.append(api.Exec(plan, ws, comms[r]))
    outs.append({o: torch.empty(og.tensors[o].shape, dtype=torch.bfloat16, device="cuda") for o in og.outputs})
st = [torch.cuda.Stream() for _ in range(2)]
th = [threading.Thread(target=lambda r=r: exs[r].run(ins, outs[r], st[r])) for r in range(2)]
[t.start() for t in th]
[t.join() for t in th]
torch.cuda.synchronize()
print("SANITIZER-RUN-OK")
"""


def _race_records(text):
    """(set of 'file:line' of each side) per race record of a racecheck report."""
    import re
    recs, cur = [], None
    for ln in text.splitlines():
        if "Race reported" in ln or "hazard" in ln.lower() and "Error" in ln:
            cur = set()
            recs.append(cur)
        if cur is not None:
            cur.update(m.group(1) + ":" + m.group(2) for m in re.finditer(r"([\w./-]+\.(?:cu|cuh|h)):(\d+)", ln))
    return [r for r in recs if r]


def _marked(loc):
    """A source line that documents a shared-memory handoff ordered by an mbarrier
    (release arrive / acquire wait), which racecheck does not model."""
    f, n = loc.rsplit(":", 1)
    path = f if os.path.isabs(f) else os.path.join(ROOT, "paper_2401_10652_b200", "csrc", os.path.basename(f))
    try:
        with open(path) as fh:
            lines = fh.read().splitlines()
    except OSError:
        return False
    i = int(n) - 1
    return any("racecheck: mbarrier handoff" in lines[k] for k in range(max(0, i - 3), min(len(lines), i + 1)))


def _skip_if_refused(r):
    # the pool may close compute-sanitizer (its wrapper then refuses with a message and
    # runs nothing): that is an unavailable tool, not a finding
    if "SANITIZER-RUN-OK" not in r.stdout and "closed on this pool" in (r.stdout + r.stderr):
        pytest.skip("compute-sanitizer refused on this pool: " + r.stderr.strip().splitlines()[0][:200])


@pytest.mark.parametrize("tool", ["racecheck", "synccheck"])
def test_racecheck_synccheck_clean(tmp_path, tool):
    """synccheck must be clean.  racecheck must report no hazard except on shared-memory
    handoffs ordered by mbarriers (arrive has release, try_wait acquire semantics; the
    tool does not model them): every reported race must have one side on a line marked
    `racecheck: mbarrier handoff` in the source."""
    san = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(san):
        pytest.skip("compute-sanitizer not found")
    script = tmp_path / "run.py"
    script.write_text(SCRIPT_SYNC % {"root": ROOT})
    r = subprocess.run([san, "--tool", tool, "--print-limit", "10000", sys.executable, str(script)],
                       capture_output=True, text=True, timeout=1500)
    _skip_if_refused(r)
    out = r.stdout + r.stderr
    dump = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(dump):
        with open(os.path.join(dump, f"sanitizer_{tool}.txt"), "w") as f:
            f.write(out)
    assert "SANITIZER-RUN-OK" in r.stdout, out[-3000:]
    if tool == "synccheck":
        assert "ERROR SUMMARY: 0 errors" in out, out[-3000:]
        return
    recs = _race_records(out)
    bad = [sorted(rc) for rc in recs if not any(_marked(loc) for loc in rc)]
    assert not bad, (len(recs), bad[:10])


def test_memcheck_clean(tmp_path):
    san = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(san):
        pytest.skip("compute-sanitizer not found")
    script = tmp_path / "run.py"
    script.write_text(SCRIPT % {"root": ROOT})
    env = dict(os.environ, PYTORCH_NO_CUDA_MEMORY_CACHING="1")
    r = subprocess.run([san, "--tool", "memcheck", "--error-exitcode", "3", "--print-limit", "10",
                        sys.executable, str(script)], capture_output=True, text=True, env=env, timeout=900)
    _skip_if_refused(r)
    assert r.returncode == 0 and "SANITIZER-RUN-OK" in r.stdout, (r.stdout[-3000:], r.stderr[-3000:])

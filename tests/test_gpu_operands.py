"""The two GEMM operand formats (common.cuh): the default fp16x2 build's range guard, and the
exact bf16x3 build (libkgq_bf16x3.so) against the oracle -- both on the GPU, through the C ABI."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O
import synth
from parity import assert_dist_close, assert_topk_ok

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)
from paper_2503_02172_b200 import Engine, KgqError, kgq  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.skipif(kgq.tensor_mmas_per_fma() != 3, reason="fp16x2 build only")
def test_fp16x2_range_guard_reports_erange():
    """An activation at or beyond the fp16 maximum (a BetaE anchor whose regularised parameter is
    1e6) makes kgq_check_errors return KGQ_ERANGE naming the format; the next check is clean.  A
    weight of magnitude >= 32 (its 2^11-scaled high plane would overflow) fails kgq_finalize."""
    N, R, d, H = 500, 8, 16, 32
    t = synth.make_tables("betae", N, R, d, hidden=H, seed=3)
    t["entity"] = t["entity"].copy()
    t["entity"][7, 3] = 1e6
    e = Engine("betae", N, R, d, hidden=H, max_batch=32, max_k=10)
    e.load_tables(t)
    a, r = synth.make_queries("1p", 20, N, R, seed=1)
    e.submit("1p", dev(a), dev(r), 10)
    e.check_errors()  # anchor 7 not used yet
    a = a.copy()
    a[5, 0] = 7
    e.submit("1p", dev(a), dev(r), 10)
    with pytest.raises(KgqError, match="fp16x2"):
        e.check_errors()
    e.check_errors()
    e.close()
    t2 = synth.make_tables("betae", N, R, d, hidden=H, seed=3)
    wk = sorted(k for k in t2 if k.startswith("W:"))[0]
    t2[wk] = t2[wk].copy()
    t2[wk][0, 0] = 40.0
    e2 = Engine("betae", N, R, d, hidden=H, max_batch=32, max_k=10)
    with pytest.raises(KgqError, match="fp16x2"):
        e2.load_tables(t2)
    e2.close()


BF16X3_CHECK = r"""
import sys
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import numpy as np, torch
import oracle as O, synth
from parity import assert_dist_close, assert_topk_ok
from paper_2503_02172_b200 import Engine, kgq
assert kgq.tensor_mmas_per_fma() == 6, kgq.LIB_PATH
N, R, d, H, B = 1000, 20, 40, 96, 37
for dist in ("kgr-init", "spread"):
    t = synth.make_tables("betae", N, R, d, hidden=H, seed=21, dist=dist)
    e = Engine("betae", N, R, d, hidden=H, max_batch=64, max_k=16)
    e.load_tables(t)
    m = O.Model("betae", t, dim=d)
    for s in synth.ALL_STRUCTURES:
        a, r = synth.make_queries(s, B, N, R, seed=synth.query_seed(7, s))
        td, ti, sd = e.submit(s, torch.from_numpy(a).cuda(), torch.from_numpy(r).cuda(), 10, shard_dist=True)
        e.check_errors()
        ref = m.scores(s, a, r)
        assert_dist_close(sd.cpu().numpy(), ref, what=f"bf16x3 {{dist}} {{s}}")
        td, ti = td.cpu().numpy(), ti.cpu().numpy()
        for b in range(B):
            assert_topk_ok(td[b], ti[b], ref[b], 10, what=f"bf16x3 {{dist}} {{s}} row {{b}}")
    e.close()
print("bf16x3 ok")
"""


def test_bf16x3_build_matches_oracle():
    """The full-range bf16x3 build (KGQ_OPERANDS=bf16x3 -> libkgq_bf16x3.so) in a fresh process:
    every BetaE structure, both input recipes, whole distance rows and top-k against the oracle."""
    env = dict(os.environ, KGQ_OPERANDS="bf16x3")
    env.pop("KGQ_LIB_PATH", None)
    code = BF16X3_CHECK.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0 and "bf16x3 ok" in p.stdout, p.stdout[-2000:] + p.stderr[-4000:]

"""GPU fault injection for the relaxed h publication (expert_fused.cu): phase-A
writers store h with plain stores and publish with relaxed counters, and a reader "settles"
its shared-memory copy — every word still carrying the armed pattern is re-read from L2
until written. On a quiet GPU the copy is almost never stale, so the debug build
(lib/libmoe_debug.so) with MOE_DEBUG_STALE_H=1 re-arms one word of every float4 of the copy
before the settle: the settle must fetch all of them again, and y must come out bit for bit
as without the injection, and within the parity bar of the oracle, in all three phase-B
layouts (merged, x beside one h buffer, segmented).

Each run is a subprocess: the library variant is chosen by MOE_LIB_PATH when the binding is
first imported."""
import json
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEBUG_LIB = os.path.join(ROOT, "paper_2512_16473_b200", "lib", "libmoe_debug.so")

CHILD = r"""
import json, os, sys
sys.path.insert(0, {root!r})
import numpy as np
import harness, oracle, inputs
import paper_2512_16473_b200 as moe
d, ff, n, K, T, out = {d}, {ff}, {n}, {K}, {T}, {out!r}
hm = harness.host_model(1, d, ff, n, K)
x, _ = harness.hidden_states(hm, T, "paper")
with harness.open_moe(hm) as m:
    m.configure(ways=n, indexes=1, warm_start=True)
    y = harness.run_decode(m, x)
    info = m.runtime_info()
ref = oracle.decode(x, hm.gates, lambda l, e: inputs.expert_weights(l, e, hm.d, hm.ff), N=1, M=n, K=K, warm_start=True)
err = max(float(np.abs(y[t, 0] - ref.y[t, 0]).max() / np.abs(ref.y[t, 0]).max()) for t in range(T))
np.save(out, y)
print(json.dumps({{"err": err, "runtime": info}}))
"""

# (d, ff, n, K): merged phase B (tiny), x beside one h buffer (single-row W2 chunks), segmented
SHAPES = {"merged": (64, 128, 8, 2), "xsep": (1024, 14336, 8, 2), "segmented": (1024, 8192, 8, 2)}


def _child(shape, stale: bool, tmp: str):
    d, ff, n, K = SHAPES[shape]
    out = os.path.join(tmp, f"y_{shape}_{int(stale)}.npy")
    env = dict(os.environ, MOE_LIB_PATH=DEBUG_LIB, MOE_DEBUG_TS="1")  # (prints the plan)
    env.pop("MOE_DEBUG_STALE_H", None)
    if stale:
        env["MOE_DEBUG_STALE_H"] = "1"
    code = CHILD.format(root=ROOT, d=d, ff=ff, n=n, K=K, T=6, out=out)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    plan = [ln for ln in r.stderr.splitlines() if ln.startswith("[moe init] fused=")][-1]
    return np.load(out), json.loads(line), plan


@pytest.mark.skipif(not os.path.exists(DEBUG_LIB), reason="debug build missing (build() makes it)")
@pytest.mark.parametrize("shape", list(SHAPES))
def test_settle_refetches_every_armed_word(shape):
    with tempfile.TemporaryDirectory() as tmp:
        y0, j0, plan = _child(shape, False, tmp)
        y1, j1, _ = _child(shape, True, tmp)
    assert j0["runtime"]["expert_path"] == "fused"
    layout = {"merged": ("merge=1", "xsep=0"), "xsep": ("merge=0", "xsep=1"), "segmented": ("merge=0", "xsep=0")}[shape]
    assert all(f in plan for f in layout), plan
    assert np.array_equal(y0.view(np.uint32), y1.view(np.uint32))
    assert j1["err"] <= 1e-4, j1

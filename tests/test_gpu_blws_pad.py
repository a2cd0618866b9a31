"""blws_svd calls that need padding (keep < r, block_lanczos.hpp:249-255).

When the deferred path fails only the keep test, it pads its own kept columns
with adapt_subspace instead of redoing the whole call on the exact path. The
leading columns of a QR depend only on the leading input columns, so the
result is the exact path's up to rounding, with the same Rng draws. The case
is the bench's C5-scale recipe at 8000^2, r = 400: the 400th Ritz value comes
out negative, so every call pads. It runs in two processes, the default and
BLWS_EXACT_PAD=1 (the redo)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import principal_angle

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASE = r"""
import sys, numpy as np, torch
sys.path.insert(0, %(root)r)
import bench
import paper_1012_0365_b200 as G
m, r = 8000, 400
Wt, Uw, Vw, sigma, U0, V0 = bench.c5_inputs(m, r, 0, m, torch.device("cuda:0"))
ctx = G.Context(0)
op = G.DenseOperator(Wt, ctx=ctx, device=True, shape=(m, m), ld=m)
warm = G.WarmStart(np.asfortranarray(Uw.cpu().numpy()), np.asfortranarray(Vw.cpu().numpy()), sigma[:r].cpu().numpy())
rng = G.Rng(11)
f0 = G.deferred_fallbacks()
res = G.blws_svd(op, warm, 2, r, rng)
np.savez(sys.argv[1], s=res.warm.sigma, u=res.warm.u, v=res.warm.v,
         flags=np.array([res.padded, res.k_raised, res.terminated_early]), nxt=np.array([rng.next_u64()], dtype=np.uint64),
         fb=np.array([G.deferred_fallbacks() - f0]))
"""


def _run(tmp_path, name, env_extra):
    env = dict(os.environ, BLWS_GRAPHS="0", **env_extra)
    out = tmp_path / f"{name}.npz"
    r = subprocess.run([sys.executable, "-c", CASE % {"root": ROOT}, str(out)], env=env, cwd=ROOT,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return dict(np.load(out))


def test_padding_from_deferred_matches_exact_redo(tmp_path):
    own = _run(tmp_path, "own", {})
    redo = _run(tmp_path, "redo", {"BLWS_EXACT_PAD": "1"})
    assert own["flags"][0] and list(own["flags"]) == list(redo["flags"])  # padded, same flags
    assert own["nxt"][0] == redo["nxt"][0]  # the same Rng draws consumed
    s1, s2 = own["s"], redo["s"]
    assert s1.shape == s2.shape
    kept = s2 > 0  # the padded columns carry sigma 0
    assert np.array_equal(kept, s1 > 0)
    assert np.abs(s1 - s2).max() <= 1e-12 * s2.max()
    k = int(kept.sum())
    assert principal_angle(own["u"][:, :k], redo["u"][:, :k]) <= 1e-9
    assert principal_angle(own["v"][:, :k], redo["v"][:, :k]) <= 1e-9
    # the padded directions: the same Gaussian draws, re-orthonormalised
    assert principal_angle(own["u"], redo["u"]) <= 1e-8 and principal_angle(own["v"], redo["v"]) <= 1e-8
    for x in (own["u"], own["v"]):
        assert np.linalg.norm(x.T @ x - np.eye(x.shape[1])) <= 1e-10

"""K8 tiled (csr_spmm_tiled_k) against scipy and, bitwise, against the gather
kernel. Run once per mode (BLWS_K8 is read once per process):
    BLWS_K8=gather python tools/probes/k8_tiled_check.py /tmp/k8_gather.npz
    BLWS_K8=tiled  python tools/probes/k8_tiled_check.py /tmp/k8_tiled.npz /tmp/k8_gather.npz
"""
import os
import sys

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1012_0365_b200 as pk  # noqa: E402

CASES = [(21000, 1500, 0.01, 9), (21000, 1500, 0.01, 55), (3001, 2999, 0.05, 33), (3001, 2999, 0.05, 31),
         (10000, 10000, 0.1, 55), (10000, 10000, 0.1, 64), (777, 20011, 0.03, 17), (14300, 500, 0.2, 50)]


def main():
    out = {}
    worst = 0.0
    for ci, (m, n, dens, b) in enumerate(CASES):
        rs = np.random.default_rng(7 * ci + b)
        a = sp.random(m, n, density=dens, format="csc", random_state=rs, data_rvs=rs.standard_normal)
        a = a.tolil()
        a[5, :] = rs.standard_normal(n)  # a dense row
        a[:, 7] = 0.0  # an empty column
        a = a.tocsc()
        a.sort_indices()
        op = pk.api.SparseOperator(m, n, a.indptr.astype(np.int64), a.indices.astype(np.int32), a.data.copy())
        left, right = rs.standard_normal((m, b)), rs.standard_normal((n, b))
        top, bot = op.apply_pair_block(left, right)
        rt, rb = a @ right, a.T @ left
        e = max(np.abs(top - rt).max() / np.abs(rt).max(), np.abs(bot - rb).max() / np.abs(rb).max())
        worst = max(worst, e)
        print(f"case {ci} {m}x{n} dens {dens} b {b}: rel err {e:.2e}", flush=True)
        out[f"top{ci}"], out[f"bot{ci}"] = top, bot
    np.savez(sys.argv[1], **out)
    assert worst <= 1e-12, worst
    if len(sys.argv) > 2:
        other = np.load(sys.argv[2])
        same = all(np.array_equal(out[k], other[k]) for k in out)
        print("bitwise equal to", sys.argv[2], ":", same)
        assert same
    print("ok")


if __name__ == "__main__":
    main()

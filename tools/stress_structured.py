"""One-off sweep of structured meshes of many sizes through every strategy against the oracle
(hex8 boxes n = 2..14 with d = 1..3, lexicographic / permuted elements / permuted nodes; tet4,
quad4 and hex27 at a few sizes): even sizes take the star patches, odd ones the host sweep.

    python tools/stress_structured.py
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle as orc  # noqa: E402  (checker)
import paper_2012_00585_b200 as fea  # noqa: E402
from paper_2012_00585_b200 import meshgen as M  # noqa: E402

orc.orc()
TOL = 1e-12
bad = 0
cases = [("hex8", n, d, perm) for n in range(2, 15) for d in (1, 2, 3) for perm in (None, "elements", "nodes")]
cases += [("tet4", n, d, perm) for n in (3, 6, 9) for d in (1, 2) for perm in (None, "nodes")]
cases += [("quad4", n, d, None) for n in (5, 17, 40) for d in (1, 2, 4)]
cases += [("hex27", n, d, None) for n in (2, 3, 4) for d in (1, 3)]
for mesh, n, d, perm in cases:
    conn, nn = M.make_mesh(mesh, n, perm)
    ed = M.element_dofs(conn, d)
    P = orc.Pattern.build(conn, nn, d)
    Kh = orc.fill_k(n, conn.shape[0], ed.shape[1])
    want = P.assemble_sequential(ed, Kh)
    ones = np.ones_like(Kh)
    want1 = P.assemble_sequential(ed, ones)
    K = torch.from_numpy(Kh).cuda()
    try:
        with fea.Plan(ed, nn * d, dofs_per_node=d) as plan:
            assert plan.assemble(K, strategy="sorted").cpu().numpy().tobytes() == want.tobytes(), "sorted"
            a = plan.assemble(K, strategy="atomic").cpu().numpy()
            assert np.all(np.abs(a - want) <= TOL * np.maximum(np.maximum(np.abs(a), np.abs(want)), 1.0)), "atomic"
            assert plan.assemble(torch.from_numpy(ones).cuda(), strategy="atomic").cpu().numpy().tobytes() == want1.tobytes(), "atomic ones"
            col, _ = plan.greedy_colouring()
            plan.set_colouring(col)
            c = plan.assemble(K, strategy="colour").cpu().numpy()
            assert c.tobytes() == P.assemble_coloured(ed, Kh, col).tobytes(), "colour"
    except Exception as e:  # noqa: BLE001
        bad += 1
        print("FAIL", mesh, n, d, perm, type(e).__name__, str(e)[:200], flush=True)
print("cases", len(cases), "failures", bad)
sys.exit(1 if bad else 0)

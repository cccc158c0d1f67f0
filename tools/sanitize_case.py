"""Small cases touching every kernel path, for compute-sanitizer (memcheck / racecheck / synccheck)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2012_00585_b200 as fea  # noqa: E402
from paper_2012_00585_b200 import meshgen as M  # noqa: E402

cases = [("quad4", 3, 1, None), ("quad4", 3, 4, "nodes"), ("hex8", 2, 3, "elements"), ("tet4", 2, 1, "nodes"),
         ("hex27", 2, 3, None), ("hex8", 3, 2, None), ("hex8", 2, 1, None)]
for mesh, n, d, perm in cases:
    conn, nn = M.make_mesh(mesh, n, perm)
    ed = M.element_dofs(conn, d)
    E, m = ed.shape
    K = fea.fill_seeded_k(E, m, 42)
    with fea.Plan(ed, nn * d, dofs_per_node=d) as plan:
        plan.set_colouring(plan.greedy_colouring()[0])
        v = None
        for s in ("sorted", "atomic", "colour", "colour_passes"):
            v = plan.assemble(K, strategy=s)
            plan.assemble(K, v, strategy=s, accumulate=True)
        plan.csr(); plan.crac()
        Kh = K.cpu().numpy()
        plan.assemble_host_batch([Kh, Kh, Kh], [np.zeros(plan.nnz) for _ in range(3)], strategy="sorted")
        rp, cs = plan.csr()
        cp, ca = plan.crac()
    for fmt, (a, b) in (("csr", (rp, cs)), ("crac", (cp, ca))):
        with fea.Plan.with_pattern(ed, nn * d, a, b, fmt) as pl:
            pl.assemble(K, strategy="sorted")
            pl.assemble(K, strategy="atomic")
    rb = (nn // 2) * d
    for kc in (False, True):
        with fea.Plan(ed, nn * d, dofs_per_node=d, row_range=(rb, nn * d), k_compact=kc) as pl:
            Kp = K[torch.from_numpy(pl.elements()).cuda()].contiguous() if kc else K
            pl.assemble(Kp, strategy="sorted")
            pl.assemble(Kp, strategy="atomic")
torch.cuda.synchronize()
print("sanitize case ok")

import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2012_00585_b200 as fea
from paper_2012_00585_b200 import meshgen as M
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
conn, nn = M.make_mesh("hex8", n, None)
ed = M.element_dofs(conn, 3)
plan = fea.Plan(ed, nn * 3, dofs_per_node=3)
K = fea.fill_seeded_k(conn.shape[0], 24, 42)
s = plan.assemble(K, strategy="sorted")
torch.cuda.synchronize()
print("sorted ok", flush=True)
a = plan.assemble(K, strategy="atomic")
torch.cuda.synchronize()
print("atomic ok", float((a - s).abs().max()), flush=True)

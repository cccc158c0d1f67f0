"""Generate tests/golden/*.npz from the UNMODIFIED reference library (oracle/_ref/libfea_ref.so).

Run in the build container (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures pin the CPU oracle and the GPU path on machines without the reference.
Every array is produced by the reference API: build_pattern (pattern.cpp:24-108), the
CracMatrix constructor (formats.cpp:21-41), greedy_colouring (colouring.cpp:24-75),
assemble_sequential / assemble_coloured_vectorized / assemble_atomic (assembly.hpp:112-195).
Inputs (meshes, seeded K) come from paper_2012_00585_b200.meshgen and oracle.fill_k; their
SHA-256 is stored so a changed generator is detected.
"""
import hashlib
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from paper_2012_00585_b200 import meshgen as M  # noqa: E402

OUT = Path(__file__).resolve().parent
SEED_K = 42

CASES = {
    "quad4_n6_d1": ("quad4", 6, 1, None),
    "quad4_n5_d2_nodeperm": ("quad4", 5, 2, "nodes"),
    "hex8_n3_d3_elemperm": ("hex8", 3, 3, "elements"),
    "tet4_n3_d1_nodeperm": ("tet4", 3, 1, "nodes"),
    "hex27_n2_d3": ("hex27", 2, 3, None),
    "hex8_n4_d1": ("hex8", 4, 1, None),
}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def make(name, conn, n_nodes, d):
    E = conn.shape[0]
    m = conn.shape[1] * d
    R = oracle.RefProblem(conn, n_nodes, d)
    rp, cs = R.pattern()
    crp, ca = R.crac()
    col, nc = R.greedy_colouring(E)
    K = oracle.fill_k(SEED_K, E, m)
    seq = R.assemble(K, "seq", "csr")
    colv = R.assemble(K, "colour-vec", "crac", threads=4, colour_of=col)
    ones = R.assemble(np.ones((E, m, m)), "atomic", "csr", threads=4)
    np.savez_compressed(OUT / f"{name}.npz", conn_sha=sha(conn), n_nodes=n_nodes, d=d,
                        k_sha=sha(K), row_ptr=rp, cols=cs, crac_ptr=crp, col_align=ca,
                        n_runs=R.n_runs, colour_of=col, n_colours=nc, values_seq=seq,
                        values_colour=colv, values_ones=ones)
    print(name, "nnz", R.nnz, "runs", R.n_runs, "colours", nc)


def main():
    for name, (mesh, n, d, perm) in CASES.items():
        conn, nn = M.make_mesh(mesh, n, perm)
        make(name, conn, nn, d)
    # the reference's own 2D p-refined numbering (build_dof_map, dof_map.cpp:24-67)
    conn, nn = oracle.ref_structured_element_nodes(4, 3, 2)
    make("refdofmap_n4_p3_d2", conn, nn, 2)
    np.save(OUT / "refdofmap_n4_p3_d2_conn.npy", conn)
    # Fig. 1 example (test_formats.cpp:31-39): CRAC arrays and lookups from the reference
    rows = [[0, 1], [0, 1], [1, 2, 4, 5], [2, 3, 4], [3, 4, 5], [1, 2, 3, 4]]
    rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    cs = np.concatenate(rows).astype(np.int64)
    R = oracle.RefProblem.from_pattern(np.zeros((0, 1), np.int64), 6, rp, cs)
    crp, ca = R.crac()
    look = np.array([[r, c, R.locate("csr", r, c), R.locate("crac", r, c)]
                     for r in range(6) for c in range(6)], np.int64)
    np.savez_compressed(OUT / "fig1.npz", row_ptr=rp, cols=cs, crac_ptr=crp, col_align=ca, lookups=look)
    print("fig1", crp, ca)


if __name__ == "__main__":
    main()

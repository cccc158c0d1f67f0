"""MSH 2.2 I/O (paper_2012_00585_b200/msh.py) — cases of the reference's test_mesh.cpp:89-172."""
import io

import numpy as np
import pytest

from paper_2012_00585_b200 import meshgen as M, msh

HEAD = "$MeshFormat\n2.2 0 8\n$EndMeshFormat\n"
NODES4 = "$Nodes\n4\n1 0 0 0\n2 1 0 0\n3 1 1 0\n4 0 1 0\n$EndNodes\n"


def test_minimal_quad_file():
    conn, nn, coords, warn, kind = msh.import_msh(HEAD + NODES4 + "$Elements\n1\n1 3 2 0 1 1 2 3 4\n$EndElements\n")
    assert conn.tolist() == [[0, 1, 2, 3]] and nn == 4 and not warn and kind == "quad4"


def test_triangle_skipped_with_warning_points_lines_ignored():
    _, _, _, warn, _ = msh.import_msh(HEAD + NODES4 + "$Elements\n2\n1 3 2 0 1 1 2 3 4\n2 2 2 0 1 1 2 3\n$EndElements\n")
    assert len(warn) == 1 and "non-quad" in warn[0]
    conn, _, _, warn, _ = msh.import_msh(HEAD + NODES4 +
                                         "$Elements\n3\n1 15 2 0 1 1\n2 1 2 0 1 1 2\n3 3 2 0 1 1 2 3 4\n$EndElements\n")
    assert conn.shape == (1, 4) and not warn


@pytest.mark.parametrize("text,msg", [
    ("$MeshFormat\n4.1 0 8\n$EndMeshFormat\n", "unsupported"),
    ("$MeshFormat\n2.2 1 8\n$EndMeshFormat\n", "unsupported"),
    (HEAD + "$Nodes\n3\n1 0 0 0\n2 1 0 0\n$EndNodes\n", "ended before declared count"),
    (HEAD + NODES4 + "$Elements\n1\n1 3 2 0 1 1 2 3 9\n$EndElements\n", "unknown node id"),
    (HEAD + NODES4 + "$Elements\n1\n1 5 2 0 1 1 2 3 4 1 2 3 4\n$EndElements\n", "volume"),
    (HEAD, "lacks"),
    (HEAD + "$Elements\n0\n$EndElements\n", "before $Nodes"),
    (HEAD + "$Nodes\n2\n1 0 0 0\n1 1 0 0\n$EndNodes\n", "duplicate node id"),
])
def test_errors(text, msg):
    with pytest.raises(msh.MshParseError, match=msg.replace("$", r"\$")):
        msh.import_msh(text)


@pytest.mark.parametrize("kind,n", [("quad4", 5), ("hex8", 3), ("tet4", 2)])
def test_round_trip(kind, n):
    conn, nn = M.make_mesh(kind, n)
    coords = msh.structured_coords(kind, n)
    out = io.StringIO()
    msh.write_msh(conn, coords, kind, out)
    c2, nn2, co2, warn, k2 = msh.import_msh(out.getvalue(), kind="auto")
    assert k2 == kind and nn2 == nn and not warn
    assert np.array_equal(c2, conn) and np.array_equal(co2, coords)


def test_cli_reads_msh(tmp_path):
    from paper_2012_00585_b200 import cli
    conn, nn = M.make_mesh("hex8", 2)
    p = tmp_path / "m.msh"
    with open(p, "w") as f:
        msh.write_msh(conn, msh.structured_coords("hex8", 2), "hex8", f)
    label, n, c2, nn2 = cli.parse_mesh(str(p))
    assert np.array_equal(c2, conn) and nn2 == nn

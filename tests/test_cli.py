"""The `fea`-compatible front end (paper_2012_00585_b200/cli.py)."""
import io

import numpy as np
import pytest

from paper_2012_00585_b200 import cli


def test_usage_errors_exit_1():
    assert cli.main(["bench", "--methods", "spin"]) == cli.EXIT_USAGE
    assert cli.main(["bench", "--methods", "bogus"]) == cli.EXIT_USAGE
    assert cli.main(["assemble", "--mesh", "missing.msh"]) == cli.EXIT_USAGE
    assert cli.main(["assemble", "--mesh", "gen:0"]) == cli.EXIT_USAGE
    assert cli.main(["assemble", "--p", "3"]) == cli.EXIT_USAGE
    assert cli.main([]) == cli.EXIT_USAGE


def test_mesh_specs():
    label, n, conn, nn = cli.parse_mesh("gen:6")
    assert conn.shape == (36, 4) and nn == 49
    _, _, conn, nn = cli.parse_mesh("hex8:3:perm-elements")
    assert conn.shape == (27, 8) and nn == 64
    _, _, conn, _ = cli.parse_mesh("tet4:2:perm-nodes")
    assert conn.shape == (48, 4)


def test_csv_schemas_match_reference():
    """bench.cpp:314-335 column order and number formats."""
    c = dict(suite="single", mesh="gen:4", n=4, p=1, d=1, dofs=25, nnz=169, method="seq", format="csr",
             threads=1, t_micros=[1.5, 2.25], t_avg=1.875, t_min=1.5, c=1.0, gamma=0.5, values_mb=0.001352)
    raw, summ = io.StringIO(), io.StringIO()
    cli.write_raw_csv([c], raw)
    cli.write_summary_csv([c], summ)
    assert raw.getvalue().splitlines() == ["suite,mesh,n,p,d,dofs,nnz,method,format,threads,run,micros",
                                           "single,gen:4,4,1,1,25,169,seq,csr,1,1,1.500",
                                           "single,gen:4,4,1,1,25,169,seq,csr,1,2,2.250"]
    assert summ.getvalue().splitlines()[1] == "single,gen:4,4,1,1,25,169,seq,csr,1,1.875,1.500,1.0000,0.500000,0.001352"


def test_matrix_market_dump():
    """formats.hpp:366-379 layout on the Fig. 1 example."""
    rows = [[0, 1], [0, 1], [1, 2, 4, 5], [2, 3, 4], [3, 4, 5], [1, 2, 3, 4]]
    rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])])
    cs = np.concatenate(rows)
    vals = np.array([1.21, 83.2, 47.1, 5.12, 6.29, 2.37, 8.34, 3.33, 9.24, 10.2, 1.17, 19.2, 13.1, 1.19,
                     16.4, 15.8, 7.36, 12.2])
    out = io.StringIO()
    cli.write_matrix_market(rp, cs, vals, out)
    lines = out.getvalue().splitlines()
    assert lines[0] == "%%MatrixMarket matrix coordinate real general"
    assert lines[1] == "6 6 18"
    assert lines[2] == "1 1 1.21" and lines[9] == "3 6 3.3300000000000001"


@pytest.mark.gpu
def test_verify_bench_assemble_on_gpu(gpu, tmp_path):
    assert cli.main(["verify", "--mesh", "hex8:4:perm-elements", "--d", "3"]) == cli.EXIT_OK
    assert cli.main(["verify", "--mesh", "tet4:3:perm-nodes"]) == cli.EXIT_OK
    out = tmp_path / "r"
    assert cli.main(["bench", "--mesh", "gen:32", "--runs", "3", "--out", str(out)]) == cli.EXIT_OK
    summ = (tmp_path / "r.summary.csv").read_text().splitlines()
    assert len(summ) == 1 + 6  # 3 methods x 2 formats
    assert cli.main(["assemble", "--mesh", "gen:2", "--dump", str(tmp_path / "a.mtx")]) == cli.EXIT_OK
    mm = (tmp_path / "a.mtx").read_text().splitlines()
    assert mm[1] == "9 9 49"  # (3n+1)^2, n = 2
    assert cli.main(["colour", "--mesh", "gen:6", "--out", str(tmp_path / "c.csv")]) == cli.EXIT_OK

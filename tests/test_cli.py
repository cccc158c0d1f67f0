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


def test_tamper_spec_parsing():
    hook = cli.parse_tamper("atomic/crac:3")
    v = np.zeros(5)
    hook("atomic/csr", v)
    assert v.sum() == 0
    hook("atomic/crac", v)
    assert v[3] == 1.0
    for bad in ("spin/crac:3", "atomic:3", "atomic/crac"):
        with pytest.raises(cli.UsageError):
            cli.parse_tamper(bad)
    assert cli.main(["verify", "--tamper", "bogus"]) == cli.EXIT_USAGE


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


@pytest.mark.gpu
def test_verify_reports_tampered_slot(gpu, capsys):
    """test_assembly.cpp:350-374: a clean run is ok; a corrupted slot of one combination makes
    verify fail (exit 2) and the first failure names that combination and the slot."""
    res = cli.verify_methods(*cli.parse_mesh("gen:4")[2:], d=2)
    assert res.ok and not res.failures and len(res.checked) == 6  # the reference: 10 (4 spin combos)

    def tamper(combo, values):
        if combo == "atomic/crac":
            values[3] += 1.0
    res = cli.verify_methods(*cli.parse_mesh("gen:4")[2:], d=1, tamper=tamper)
    assert not res.ok and len(res.failures) >= 1
    assert "atomic/crac" in res.failures[0] and "values[3]" in res.failures[0]
    capsys.readouterr()
    assert cli.main(["verify", "--mesh", "gen:4", "--tamper", "colour-vec/csr:7:0.5"]) == cli.EXIT_VERIFY_FAILED
    outp = capsys.readouterr().out
    assert "verify: FAIL colour-vec/csr: values[7]" in outp and "combinations: 6" in outp


@pytest.mark.gpu
@pytest.mark.parametrize("mesh,d", [("gen:5", 2), ("hex8:3:perm-elements", 3), ("tet4:3:perm-nodes", 1)])
def test_dump_and_bench_csv_match_oracle(gpu, orc, tmp_path, mesh, d):
    """`assemble --dump` (fea_main.cpp:239-253: ones supplier, assemble_sequential, Matrix Market
    formats.hpp:366-379) is byte-identical to the oracle's matrix through the same writer; the
    bench CSV's dofs / nnz / storage factor equal the oracle's pattern (bench.cpp:100-113)."""
    import io
    _, _, conn, nn = cli.parse_mesh(mesh)
    from paper_2012_00585_b200 import meshgen as M
    ed = M.element_dofs(conn, d)
    P = orc.Pattern.build(conn, nn, d)
    want = P.assemble_sequential(ed, np.ones((ed.shape[0], ed.shape[1], ed.shape[1])))
    rp, cs = P.arrays()
    buf = io.StringIO()
    cli.write_matrix_market(rp, cs, want, buf)
    path = tmp_path / "a.mtx"
    assert cli.main(["assemble", "--mesh", mesh, "--d", str(d), "--dump", str(path)]) == cli.EXIT_OK
    assert path.read_text() == buf.getvalue()
    out = tmp_path / "b"
    assert cli.main(["bench", "--mesh", mesh, "--d", str(d), "--runs", "2", "--out", str(out)]) == cli.EXIT_OK
    lines = (tmp_path / "b.summary.csv").read_text().splitlines()
    hdr = lines[0].split(",")
    for line in lines[1:]:
        row = dict(zip(hdr, line.split(",")))
        assert int(row["dofs"]) == P.n_rows and int(row["nnz"]) == P.nnz
        assert float(row["gamma"]) == pytest.approx((2 * P.n_runs + 2) / P.nnz, abs=1e-6)
        assert float(row["values_mb"]) == pytest.approx(8.0 * P.nnz / 1e6, abs=1e-6)
    raw = (tmp_path / "b.raw.csv").read_text().splitlines()
    assert len(raw) == 1 + 6 * 2 and all(float(r.split(",")[-1]) > 0 for r in raw[1:])

"""CPU tests of the host-side pieces: CSV/JSON I/O rules (io.cpp), the named
generator families (generators.cpp, test_harness.cpp:56-133, :243-260) and the
CLI's argument / input validation that runs before any device work
(test_cli.cpp:122-147)."""
import numpy as np
import pytest

from paper_2506_14780_b200 import cli
from paper_2506_14780_b200 import generators as G
from paper_2506_14780_b200 import io as sio


def test_format_double_round_trips_bitwise():
    r = np.random.default_rng(0)
    vals = np.concatenate([r.standard_normal(200) * 10.0 ** r.integers(-300, 300, 200), [0.0, -0.0, 1 / 3]])
    for v in vals:
        assert float(sio.format_double(v)) == v


def test_csv_header_and_errors(tmp_path):
    p = tmp_path / "m.csv"
    p.write_text("a,b\n1,2\n3,4\r\n\n5, 6 \n")
    m = sio.read_csv_matrix(str(p))
    assert m.shape == (3, 2) and m[2, 1] == 6.0 and m.flags.f_contiguous
    bad = tmp_path / "bad.csv"
    bad.write_text("0,1\n2,x\n")
    with pytest.raises(sio.CsvError, match="bad.csv:2:2: not a number: 'x'"):
        sio.read_csv_matrix(str(bad))
    inf = tmp_path / "inf.csv"
    inf.write_text("0,1\n2,inf\n")
    with pytest.raises(sio.CsvError, match="inf.csv:2:2: non-finite value rejected"):
        sio.read_csv_matrix(str(inf))
    ragged = tmp_path / "ragged.csv"
    ragged.write_text("0,1\n2\n")
    with pytest.raises(sio.CsvError, match="inconsistent column count"):
        sio.read_csv_matrix(str(ragged))
    empty = tmp_path / "empty.csv"
    empty.write_text("x,y\n")
    with pytest.raises(sio.CsvError, match="no data rows"):
        sio.read_csv_matrix(str(empty))
    with pytest.raises(sio.CsvError, match="cannot open file"):
        sio.read_csv_matrix(str(tmp_path / "missing.csv"))
    over = tmp_path / "over.csv"
    over.write_text("1\n1e400\n")  # (on line 1 it would be taken for a header)
    with pytest.raises(sio.CsvError, match="not a number"):
        sio.read_csv_matrix(str(over))
    trailing = tmp_path / "trailing.csv"
    trailing.write_text("0,0,0\n1,2,\n")
    with pytest.raises(sio.CsvError, match="2:3: not a number: ''"):
        sio.read_csv_matrix(str(trailing))


def test_point_cloud_weights(tmp_path):
    p = tmp_path / "pc.csv"
    p.write_text("x,y,weight\n0,0,1\n1,1,3\n")
    pts, w, ren = sio.read_point_cloud(str(p))
    assert pts.shape == (2, 2) and ren and np.allclose(w, [0.25, 0.75])
    q = tmp_path / "pc2.csv"
    q.write_text("0,0,1\n1,1,3\n")  # no header: pure coordinates
    pts, w, ren = sio.read_point_cloud(str(q))
    assert pts.shape == (2, 3) and not ren and np.all(w == 0.5)
    z = tmp_path / "pc3.csv"
    z.write_text("x,weight\n0,1\n1,0\n")
    with pytest.raises(sio.CsvError, match="pc3.csv:3:2: weights must be strictly positive"):
        sio.read_point_cloud(str(z))
    v = tmp_path / "v.csv"
    v.write_text("1,2,3\n")
    assert np.array_equal(sio.read_csv_vector(str(v)), [1.0, 2.0, 3.0])


def test_writers(tmp_path):
    sio.write_potentials_csv(str(tmp_path / "p.csv"), [0.1, 0.2], [1 / 3])
    assert (tmp_path / "p.csv").read_text() == ("which,index,value\nf,0,0.10000000000000001\n"
                                                "f,1,0.20000000000000001\ng,0,0.33333333333333331\n")
    rep = {"epsilon": 0.5, "rho": np.array([0.25, 0.125]), "hessian_eigs_low": np.array([1.5, 1.75])}
    js = sio.spectrum_report_to_json(rep, 2)
    assert js == ('{\n  "epsilon": 0.5,\n  "k": 2,\n  "rho": [0.25, 0.125],\n'
                  '  "hessian_eigs_low": [1.5, 1.75]\n}\n')
    import json
    rep["vectors_f"] = np.eye(2)
    rep["vectors_g"] = np.ones((3, 2))
    back = json.loads(sio.spectrum_report_to_json(rep, 2))
    assert back["vectors_g"] == [[1.0, 1.0, 1.0], [1.0, 1.0, 1.0]]


def test_gaussian_cloud_determinism_and_validation():  # test_harness.cpp:56-82
    x, w = G.gaussian_cloud(200, (0.0, 0.0), np.eye(2), 1)
    y, _ = G.gaussian_cloud(400, (4.0, 4.0), [[1.0, -0.8], [-0.8, 1.0]], 2)
    assert x.shape == (200, 2) and y.shape == (400, 2) and w[0] == 1.0 / 200
    x2, _ = G.gaussian_cloud(200, (0.0, 0.0), np.eye(2), 1)
    assert np.array_equal(x, x2)
    with pytest.raises(ValueError, match="positive definite"):
        G.gaussian_cloud(10, (0.0, 0.0), [[1.0, 2.0], [2.0, 1.0]], 1)
    big, _ = G.gaussian_cloud(20000, (4.0, 4.0), [[1.0, -0.8], [-0.8, 1.0]], 3)
    assert np.all(np.abs(big.mean(axis=0) - 4.0) <= 0.05)


def test_two_moons_and_annulus_geometry():  # test_harness.cpp:84-112
    (up, _), (lo, _) = G.two_moons(64, 0.0, 5)
    assert np.all(np.abs(np.hypot(up[:, 0], up[:, 1]) - 1.0) <= 1e-12) and np.all(up[:, 1] >= -1e-12)
    assert np.all(np.abs(np.hypot(lo[:, 0] - 1.0, lo[:, 1] - 0.5) - 1.0) <= 1e-12)
    (ann, _), (sq, _) = G.annulus_and_square(256, 128, 0.5, 1.0, 2.0, 6)
    r = np.hypot(ann[:, 0], ann[:, 1])
    assert np.all(r >= 0.5) and np.all(r <= 1.0) and np.all(np.abs(sq) <= 1.0)
    with pytest.raises(ValueError, match="r_in < r_out"):
        G.annulus_and_square(10, 10, 1.0, 0.5, 2.0, 6)


def test_make_instance_families():  # test_harness.cpp:243-260
    for fam in ("gauss2d", "two_moons", "annulus_square"):
        a = G.make_instance(fam, 30, 40, seed=4)
        b = G.make_instance(fam, 30, 40, seed=4)
        assert a[0].shape == (30, 2) and a[2].shape == (40, 2)
        assert all(np.array_equal(p, q) for p, q in zip(a, b))
    with pytest.raises(ValueError, match="unknown family 'nope'"):
        G.make_instance("nope", 3, 3)


def test_cli_input_validation(tmp_path, capsys):  # test_cli.cpp:122-147
    assert cli.main(["solve", "--epsilon", "1.0"]) == 1
    assert "exactly one of --synthetic, --points, --cost is required" in capsys.readouterr().err
    bad = tmp_path / "bad.csv"
    bad.write_text("0,1\n2,x\n")
    assert cli.main(["solve", "--cost", str(bad), "--epsilon", "1.0"]) == 1
    assert "bad.csv:2:2" in capsys.readouterr().err
    assert cli.main(["anneal", "--synthetic", "gauss2d", "--schedule", "0.1", "--warm", "hot"]) == 1
    assert "--warm must be none, potentials or spectral" in capsys.readouterr().err

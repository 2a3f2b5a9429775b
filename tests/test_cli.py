"""Command line (reference cli.py): the host-side
argument handling and exit codes on CPU; select / deform / bench / metrics
through the device path on the GPU, checked against the oracle and against
the package API they wrap."""

import numpy as np
import pytest

from conftest import import_reference, reference_available
from paper_2004_04817_b200 import cli
from paper_2004_04817_b200 import deformers as D
from paper_2004_04817_b200 import meshio as M
from paper_2004_04817_b200 import workloads as W

BEND = ["--deform-mode", "bend-twist", "--b", "1.0", "--theta-m", "30", "--x0", "0.25"]


@pytest.fixture(scope="module")
def wing(tmp_path_factory):
    """600 wing-surface boundary nodes + 400 volume nodes as an MDK1 mesh,
    and the wing's own displacement field as an MDK1-DISP file."""
    wl = W.random_wing(600, 400, seed=0, m=4)
    nodes = np.vstack([wl.points, wl.volume])
    mesh = M.Mesh(nodes=nodes, boundary=np.arange(600), cells=[])
    d = tmp_path_factory.mktemp("cli")
    (d / "wing.mdk1").write_text(M.write_mesh(mesh))
    (d / "wing.disp").write_text(M.write_displacements(wl.disp, mesh.boundary))
    return d / "wing.mdk1", d / "wing.disp", wl


# ------------------------------------------------------------------ CPU
def test_deformers_known_values():
    bt = D.BendTwistParams(b=2.0, theta_m=30.0, x0=0.5)
    p = np.array([[1.5, 0.0, 2.0]])  # tip: sin(pi/2) = 1 -> 30 deg, bend 0.05 * 2
    d = D.bend_twist(p, bt)
    c, s = np.cos(np.radians(30.0)), np.sin(np.radians(30.0))
    assert np.allclose(d[0], [c * 1.0 - 1.0, s * 1.0 + 0.1, 0.0], rtol=0, atol=1e-15)
    assert D.bend_twist(p[0], bt).shape == (3,)
    ss = D.SpanSineParams(b=1.0, c=0.5)
    assert D.span_sine(np.array([0.0, 0.0, 1.0 / 16]), ss)[1] == pytest.approx(0.15 / 256)
    with pytest.raises(ValueError):
        D.BendTwistParams(b=0.0, theta_m=1.0)
    with pytest.raises(D.SourceMismatchError):
        D.prescribe(np.zeros((3, 3)))
    with pytest.raises(D.SourceMismatchError):
        D.prescribe(np.zeros((3, 3)), field=np.zeros((2, 3)))


@pytest.mark.skipif(not reference_available(), reason="reference not mounted")
def test_deformers_bitwise_equal_reference(rng):
    R = import_reference()
    from rbfdeform import deformers as RD

    pts = rng.normal(size=(500, 3))
    for ours, theirs in ((D.BendTwistParams(1.3, 25.0, 0.2, -0.1), RD.BendTwistParams(1.3, 25.0, 0.2, -0.1)),):
        assert np.array_equal(D.bend_twist(pts, ours), RD.bend_twist(pts, theirs))
    assert np.array_equal(D.span_sine(pts, D.SpanSineParams(2.0, 0.7)),
                          RD.span_sine(pts, RD.SpanSineParams(2.0, 0.7)))
    assert R is not None


def test_usage_and_source_errors_exit_codes(wing, tmp_path, capsys):
    mesh, disp, _ = wing
    with pytest.raises(SystemExit) as e:
        cli.main(["select", *BEND])
    assert e.value.code == 2
    assert cli.main(["select", "--mesh", str(tmp_path / "nope.mdk1"), *BEND]) == 1
    assert cli.main(["select", "--mesh", str(mesh)]) == 1  # no displacement source
    assert cli.main(["select", "--mesh", str(mesh), "--disp", str(disp), *BEND]) == 1  # two
    assert cli.main(["select", "--mesh", str(mesh), "--deform-mode", "bend-twist"]) == 1  # no --b
    assert cli.main(["select", "--mesh", str(mesh), "--deform-mode", "span-sine", "--b", "1"]) == 1
    assert cli.main(["select", "--mesh", str(mesh), "--disp", str(disp), "--algorithm", "gcb",
                     "--m", "x"]) == 1
    assert cli.main(["bench", "--mesh", str(mesh), "--disp", str(disp), "--m-list", ",",
                     "--out", str(tmp_path / "b.csv")]) == 1
    assert cli.main(["bench", "--mesh", str(mesh), "--disp", str(disp), "--m-list", "a",
                     "--out", str(tmp_path / "b.csv")]) == 1
    assert cli.main(["make-wing", "--out", str(tmp_path / "w.mdk1")]) == 1  # not registered
    assert "error:" in capsys.readouterr().err


def test_parser_matches_reference_flags():
    if not reference_available():
        pytest.skip("reference not mounted")
    import_reference()
    from rbfdeform import cli as RC

    def flags(parser):
        sub = next(a for a in parser._actions if a.dest == "command")
        return {name: sorted((tuple(a.option_strings), a.default, a.required) for a in p._actions
                             if a.option_strings and a.dest != "help")
                for name, p in sub.choices.items()}

    ours, theirs = flags(cli.build_parser()), flags(RC.build_parser())
    assert ours.keys() == theirs.keys()
    for name in ours:
        assert [f[0] for f in ours[name]] == [f[0] for f in theirs[name]], name
        assert [(f[1], f[2]) for f in ours[name]] == [(f[1], f[2]) for f in theirs[name]], name


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
def test_select_matches_oracle_and_api(cuda, wing, tmp_path, capsys):
    import rbf_oracle as O

    mesh, disp, wl = wing
    sup, hist = tmp_path / "s.csv", tmp_path / "h.csv"
    args = ["select", "--mesh", str(mesh), "--disp", str(disp), "--radius", "2.0", "--tol",
            repr(wl.tol), "--algorithm", "gcb", "--m", "4", "--supports-out", str(sup),
            "--history", str(hist)]
    assert cli.main(args) == 0
    out = capsys.readouterr().out
    ref = O.select(wl.points, wl.disp, 2.0, wl.tol, 600, 4, 0)
    s = M.read_supports_csv(sup.read_text())
    assert np.array_equal(s.nodes, ref["seq"])
    assert np.abs(s.weights - ref["weights"]).max() <= 1e-9 * np.abs(ref["weights"]).max()
    assert f"supports: {len(ref['seq'])} of 600 boundary nodes (m=4)" in out
    assert "converged: true" in out
    h = M.read_history_csv(hist.read_text())
    assert [r.node for r in h.records] == [r.node for r in cuda.gcb_select(
        cuda.BoundarySet(np.arange(600), wl.points, wl.disp),
        cuda.SelectionConfig(radius=2.0, tol=wl.tol, max_supports=600, m=4)).history.records]
    # greedy == gcb m = 1 (reference tests/test_cli.py:63-74), timing columns stripped
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    base = ["select", "--mesh", str(mesh), "--disp", str(disp), "--radius", "2.0", "--tol", "1e-5"]
    assert cli.main(base + ["--history", str(a)]) == 0
    assert cli.main(base + ["--algorithm", "gcb", "--m", "1", "--history", str(b)]) == 0

    def strip(t):
        return "\n".join(",".join(ln.split(",")[:-2]) for ln in t.splitlines())

    assert strip(a.read_text()) == strip(b.read_text())
    # huge tolerance: seeds only; unconverged without a cap -> 1; with a cap -> 0
    assert cli.main(base[:-2] + ["--tol", "1e9"]) == 0
    assert "supports: 3 of" in capsys.readouterr().out
    assert cli.main(base[:-2] + ["--tol", "1e-15", "--max-supports", "10"]) == 0
    assert cli.main(base[:-2] + ["--tol", "1e-15", "--radius", "0.05"]) in (0, 1)
    assert cli.main(base + ["--algorithm", "gcb", "--m", "auto"]) == 0
    assert "(m=" in capsys.readouterr().out


@pytest.mark.gpu
def test_deform_zero_and_prescribed(cuda, wing, tmp_path):
    mesh_path, disp, wl = wing
    mesh = M.read_mesh(mesh_path.read_text())
    zero = tmp_path / "zero.disp"
    zero.write_text(M.write_displacements(np.zeros((600, 3)), mesh.boundary))
    out = tmp_path / "d.mdk1"
    assert cli.main(["deform", "--mesh", str(mesh_path), "--disp", str(zero), "--radius", "2.0",
                     "--out", str(out)]) == 0
    assert out.read_text() == M.write_mesh(mesh)
    # prescribed field: boundary lands on target, volume equals deform_points of the support
    sup = tmp_path / "s.csv"
    assert cli.main(["deform", "--mesh", str(mesh_path), "--disp", str(disp), "--radius", "2.0",
                     "--tol", "1e-7", "--out", str(out), "--supports-out", str(sup)]) == 0
    after = M.read_mesh(out.read_text())
    assert np.abs(after.boundary_points() - (wl.points + wl.disp)).max() <= 2e-7
    s = M.read_supports_csv(sup.read_text())
    assert np.array_equal(after.nodes, M.read_mesh(M.write_mesh(M.Mesh(
        nodes=cuda.deform_points(mesh.nodes, s, 2.0), boundary=mesh.boundary, cells=[]))).nodes)
    # reuse a supports file
    out2 = tmp_path / "d2.mdk1"
    assert cli.main(["deform", "--mesh", str(mesh_path), "--disp", str(disp), "--radius", "2.0",
                     "--supports", str(sup), "--out", str(out2)]) == 0
    assert out2.read_text() == out.read_text()


@pytest.mark.gpu
def test_bench_rows_and_metrics(cuda, wing, tmp_path):
    mesh, disp, wl = wing
    out = tmp_path / "bench.csv"
    assert cli.main(["bench", "--mesh", str(mesh), "--disp", str(disp), "--radius", "2.0", "--tol",
                     repr(wl.tol), "--m-list", "1,4", "--out", str(out)]) == 0
    lines = out.read_text().splitlines()
    assert lines[0] == cli.BENCH_HEADER and len(lines) == 3
    b = cuda.BoundarySet(np.arange(600), wl.points, wl.disp)
    for line, m in zip(lines[1:], (1, 4)):
        row = line.split(",")
        res = cuda.gcb_select(b, cuda.SelectionConfig(radius=2.0, tol=wl.tol, max_supports=600, m=m))
        assert [int(row[0]), int(row[1]), row[2], int(row[3]), int(row[4])] == [
            m, len(res.support), str(res.converged).lower(), len(res.history.records),
            cuda.error_stage_cost(res.history)]
        assert all(float(v) >= 0 for v in row[5:])
    # KL of identical sets is 0; random baseline is farther
    s1 = tmp_path / "one.csv"
    assert cli.main(["select", "--mesh", str(mesh), "--disp", str(disp), "--radius", "2.0",
                     "--max-supports", "40", "--tol", "1e-12", "--supports-out", str(s1)]) == 0
    s2 = tmp_path / "two.csv"
    s2.write_text(s1.read_text())
    rep = tmp_path / "kl.csv"
    cli.QUALITY_REPORT = lambda cells, nodes: type("Q", (), dict(q=np.zeros(0), q_min=0.0, q_mean=0.0,
                                                                     histogram=np.zeros(20)))()
    try:
        assert cli.main(["metrics", "--mesh", str(mesh), "--supports", str(s1), str(s2), "--random",
                         "40:123", "--radius", "2.0", "--report", str(rep)]) == 0
    finally:
        cli.QUALITY_REPORT = None
    kl = {ln.split(",")[1]: float(ln.split(",")[2]) for ln in rep.read_text().splitlines()
          if ln.startswith("kl,")}
    assert kl["one||two"] == 0.0 and kl["two||one"] == 0.0
    assert kl["one||random1"] > 0.0

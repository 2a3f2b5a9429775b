"""Mesh / result I/O (reference meshio.py): canonical writers byte-identical
to the reference's output (golden files written by the reference), readers
with the reference's errors and line numbers, the native codec agreeing
with the reference-grammar path on every input. Host code: runs on CPU."""

import io

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from conftest import GOLDEN, load_golden
from paper_2004_04817_b200 import meshio as M
from paper_2004_04817_b200.errors import (
    DuplicateNodeError,
    InvariantViolationError,
    MissingNodeError,
    ParseError,
    RBFDeformError,
)

MINI = "MDK1\nNODES 3\n0 0 0\n1 0 0\n0 1 0\nBOUNDARY 3\n0\n1\n2\nCELLS 0\n"


def both(text):
    """(native result or None, reference-grammar result): they must agree."""
    return M._read_mesh_native(text), M._read_mesh_py(text)


def same_mesh(a, b):
    return (np.array_equal(a.nodes, b.nodes) and np.array_equal(a.boundary, b.boundary)
            and len(a.cells) == len(b.cells)
            and all(np.array_equal(x, y) for x, y in zip(a.cells, b.cells)))


# ----------------------------------------------------------- golden bytes
def test_writers_byte_identical_to_reference_golden():
    g = load_golden("meshio_values")
    mesh = M.Mesh(nodes=g["nodes"], boundary=g["boundary"],
                  cells=[np.array([0, 1, 2]), np.array([3, 4, 5, 6])])
    assert M.write_mesh(mesh) == (GOLDEN / "meshio_mesh.mdk1").read_text()
    assert M.write_displacements(g["disp"], mesh.boundary) == (GOLDEN / "meshio_disp.mdk1").read_text()
    from paper_2004_04817_b200 import SupportSet

    sup = SupportSet(g["sup_nodes"], g["sup_points"], g["sup_weights"])
    assert M.write_supports_csv(sup) == (GOLDEN / "meshio_supports.csv").read_text()
    hist = M.read_history_csv((GOLDEN / "meshio_history.csv").read_text())
    assert M.write_history_csv(hist) == (GOLDEN / "meshio_history.csv").read_text()


def test_readers_recover_golden_values_exactly():
    g = load_golden("meshio_values")
    mesh = M.read_mesh(io.StringIO((GOLDEN / "meshio_mesh.mdk1").read_text()))
    assert np.array_equal(mesh.nodes, g["nodes"])      # includes -0 and a subnormal
    assert np.array_equal(mesh.boundary, np.sort(g["boundary"]))
    d = M.read_displacements((GOLDEN / "meshio_disp.mdk1").read_text(), mesh.boundary)
    assert np.array_equal(d, g["disp"])
    s = M.read_supports_csv((GOLDEN / "meshio_supports.csv").read_text())
    assert np.array_equal(s.points, g["sup_points"]) and np.array_equal(s.weights, g["sup_weights"])


# ------------------------------------------------------------ read_mesh
def test_minimal_and_comments():
    m = M.read_mesh(io.StringIO(MINI))
    assert (m.n_nodes, m.n_boundary, m.cells) == (3, 3, [])
    m = M.read_mesh(MINI.replace("NODES 3", "NODES 3  # count") + "\n# end\n\n")
    assert m.n_nodes == 3
    nat, ref = both(MINI)
    assert nat is not None and same_mesh(nat, ref)


def test_cells_and_sorted_boundary():
    m = M.read_mesh(MINI.replace("CELLS 0", "CELLS 2\n3 0 1 2\n3 2 1 0"))
    assert [c.tolist() for c in m.cells] == [[0, 1, 2], [2, 1, 0]]
    m = M.read_mesh(MINI.replace("BOUNDARY 3\n0\n1\n2", "BOUNDARY 3\n2\n0\n1"))
    assert m.boundary.tolist() == [0, 1, 2]


@pytest.mark.parametrize("text,exc,line", [
    ("MDK9\n", ParseError, 1),
    ("MDK1\nNODES 2\n0 0 0\n", ParseError, 4),
    ("MDK1\nNODES 1\n0 0\n", ParseError, 3),
    ("MDK1\nNODES 1\n0 0 x\nBOUNDARY 0\nCELLS 0\n", ParseError, 3),
    ("MDK1\nNODES 1\n0 0 nan\nBOUNDARY 0\nCELLS 0\n", InvariantViolationError, 3),
    ("MDK1\nNODES 1\n0 0 1e400\nBOUNDARY 0\nCELLS 0\n", InvariantViolationError, 3),
    (MINI.replace("BOUNDARY 3\n0\n1\n2", "BOUNDARY 3\n0\n1\n7"), InvariantViolationError, 9),
    (MINI.replace("BOUNDARY 3\n0\n1\n2", "BOUNDARY 3\n0\n1\n1"), InvariantViolationError, 9),
    (MINI.replace("CELLS 0", "CELLS 1\n5 0 1 2 0 1"), InvariantViolationError, 11),
    (MINI.replace("CELLS 0", "CELLS 1\n3 0 1 9"), InvariantViolationError, 11),
    (MINI.replace("CELLS 0", "CELLS 1\n4 0 1 2"), ParseError, 11),
    (MINI + "EXTRA\n", ParseError, 11),
    ("MDK1\nNODES -1\n", ParseError, 2),
])
def test_errors_name_their_line(text, exc, line):
    with pytest.raises(exc) as err:
        M.read_mesh(text)
    assert type(err.value) is exc and err.value.line == line
    assert M._read_mesh_native(text) is None


def test_out_of_range_message_names_index():
    with pytest.raises(InvariantViolationError) as err:
        M.read_mesh(MINI.replace("BOUNDARY 3\n0\n1\n2", "BOUNDARY 3\n0\n1\n7"))
    assert "7" in str(err.value)


@pytest.mark.parametrize("token,value", [
    ("1_0", 10.0), ("+.5", 0.5), ("5.", 5.0), ("-0", -0.0), ("1E3", 1000.0), ("1e-320", 1e-320),
    (" 1", 1.0), ("0x10", None), ("inf", None), ("--1", None),
])
def test_native_and_reference_grammar_agree(token, value):
    text = f"MDK1\nNODES 1\n0 0 {token}\nBOUNDARY 1\n0\nCELLS 0\n"
    if value is None:
        with pytest.raises(ParseError):
            M.read_mesh(text)
        return
    m = M.read_mesh(text)
    assert m.nodes[0, 2] == value and np.signbit(m.nodes[0, 2]) == np.signbit(value)


@settings(max_examples=80, deadline=None)
@given(st.text(max_size=300))
def test_never_crashes_on_junk(text):
    try:
        M.read_mesh(text)
    except RBFDeformError:
        pass


@settings(max_examples=60, deadline=None)
@given(st.lists(st.tuples(st.floats(allow_nan=False, allow_infinity=False, width=64),
                          st.floats(allow_nan=False, allow_infinity=False, width=64),
                          st.floats(allow_nan=False, allow_infinity=False, width=64)),
                min_size=1, max_size=30),
       st.sampled_from(["", "  ", "\t", " # c"]))
def test_native_equals_reference_grammar_on_random_meshes(rows, pad):
    nodes = np.array(rows, dtype=float)
    mesh = M.Mesh(nodes=nodes, boundary=np.arange(min(3, len(nodes))))
    text = M.write_mesh(mesh).replace("\n", pad + "\n")
    nat, ref = both(text)
    assert same_mesh(ref, mesh)
    if nat is not None:
        assert same_mesh(nat, ref)


def test_large_mesh_native_round_trip():
    rng = np.random.default_rng(5)
    nodes = rng.normal(size=(200_000, 3)) * 10.0 ** rng.integers(-8, 8, size=(200_000, 1))
    mesh = M.Mesh(nodes=nodes, boundary=rng.choice(200_000, 5000, replace=False),
                  cells=[np.array([0, 1, 2]), np.array([3, 4, 5, 6])])
    text = M.write_mesh(mesh)
    back = M._read_mesh_native(text)
    assert back is not None and same_mesh(back, mesh)
    assert M.write_mesh(back) == text
    head = "\n".join(text.splitlines()[:2002]) + "\n"  # the reference-grammar path on a prefix
    assert np.array_equal(M._read_mesh_py(head.replace("NODES 200000", "NODES 2000")
                                          + "BOUNDARY 0\nCELLS 0\n").nodes, nodes[:2000])


def test_canonical_round_trip_bytes_and_newlines(rng):
    mesh = M.Mesh(nodes=rng.normal(size=(5, 3)), boundary=np.array([0, 2, 4]),
                  cells=[np.array([0, 1, 2]), np.array([1, 2, 3, 4])])
    text = M.write_mesh(mesh)
    assert M.write_mesh(M.read_mesh(text)) == text and "\r" not in text
    assert M.write_mesh(M.read_mesh(MINI)) == MINI


# --------------------------------------------------------- displacements
def test_displacements_golden_and_errors():
    text = "MDK1-DISP\n2 0.5 0 0\n0 1 2 3\n5 -1 0 0.25\n"
    assert M.read_displacements(io.StringIO(text), np.array([0, 2, 5])).tolist() == \
        [[1, 2, 3], [0.5, 0, 0], [-1, 0, 0.25]]
    assert M.read_displacements(io.StringIO("MDK1-DISP\n"), np.array([], int)).shape == (0, 3)
    with pytest.raises(DuplicateNodeError):
        M.read_displacements("MDK1-DISP\n0 1 0 0\n0 2 0 0\n", np.array([0, 1]))
    with pytest.raises(MissingNodeError):
        M.read_displacements("MDK1-DISP\n0 1 0 0\n", np.array([0, 1]))
    with pytest.raises(ParseError) as err:
        M.read_displacements("MDK1-DISP\n0 1 0 0\n7 1 0 0\n", np.array([0, 1]))
    assert err.value.line == 3
    with pytest.raises(ParseError):
        M.read_displacements("MDK1-DISP\n0 1 0\n", np.array([0]))


def test_displacements_round_trip(rng):
    b = np.sort(rng.choice(10_000, 3000, replace=False))
    d = rng.normal(size=(3000, 3)) * 1e-3
    text = M.write_displacements(d, b)
    assert np.array_equal(M.read_displacements(text, b), d)
    assert np.array_equal(M._read_disp_py(text, b), d)


# ----------------------------------------------------------------- CSVs
def test_history_and_supports_csv(rng):
    from paper_2004_04817_b200 import IterationRecord, SelectionHistory, SupportSet

    h = SelectionHistory()
    assert M.write_history_csv(h) == M.HISTORY_HEADER + "\n"
    h.records.append(IterationRecord(3, 0, 7, 0.25, 10, 10, 1e-6, 0.0))
    h.final_sweep = IterationRecord(5, -1, 2, 1e-9, 30, 40, 2e-6, 0.0)
    back = M.read_history_csv(M.write_history_csv(h))
    assert back.records[0] == h.records[0] and back.final_sweep == h.final_sweep
    with pytest.raises(ParseError):
        M.read_history_csv("nope\n")
    with pytest.raises(ParseError):
        M.read_history_csv(M.HISTORY_HEADER + "\n1,2,3\n")
    s = SupportSet(np.array([4, 9]), rng.normal(size=(2, 3)), rng.normal(size=(2, 3)))
    back = M.read_supports_csv(M.write_supports_csv(s))
    assert np.array_equal(back.nodes, s.nodes) and np.array_equal(back.points, s.points)
    assert np.array_equal(back.weights, s.weights)
    with pytest.raises(ParseError):
        M.read_supports_csv(M.SUPPORTS_HEADER + "\n1,2\n")


def test_npz_binary_path(tmp_path, rng):
    mesh = M.Mesh(nodes=rng.normal(size=(50, 3)), boundary=np.array([3, 1]),
                  cells=[np.array([0, 1, 2]), np.array([1, 2, 3, 4])])
    M.save_mesh_npz(tmp_path / "m.npz", mesh)
    back = M.load_mesh_npz(tmp_path / "m.npz")
    assert same_mesh(back, mesh)

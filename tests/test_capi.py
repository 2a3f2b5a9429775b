"""The C-ABI library builds, loads without a GPU, exports every symbol that
include/rbf_b200.h declares, and its struct layouts match the ctypes
mirror in paper_2004_04817_b200/_native.py. No compute calls here."""

import ctypes
import re
import subprocess

import pytest

from conftest import REPO
from paper_2004_04817_b200 import _native as N

HEADER = REPO / "include" / "rbf_b200.h"


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"RBF_API\s+[\w\s\*]+?\b(rbf_\w+)\s*\(", text)))


def test_header_declares_the_abi():
    names = declared_functions()
    assert "rbf_gcb_run" in names and "rbf_eval" in names and len(names) >= 11


def test_library_loads_and_exports_every_declared_symbol():
    lib = N.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
    bound = {s[0] for s in N.SIGNATURES}
    assert bound == set(declared_functions())
    assert lib.rbf_abi_version() == 1


def test_symbols_visible_in_dynamic_table():
    out = subprocess.run(["nm", "-D", "--defined-only", str(N.lib_path())],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (rbf_\w+)", out))
    assert set(declared_functions()) <= exported


def test_library_targets_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(N.lib_path())],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def test_struct_layout_matches_ctypes(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "rbf_b200.h"\n'
        "#define P(T, f) printf(#T \".\" #f \" %zu\\n\", offsetof(T, f));\n"
        "int main(void){\n"
        'printf("rbf_gcb_args %zu\\n", sizeof(rbf_gcb_args));\n'
        'printf("rbf_gcb_state %zu\\n", sizeof(rbf_gcb_state));\n'
        'printf("rbf_gcb_record %zu\\n", sizeof(rbf_gcb_record));\n'
        + "".join(f"P(rbf_gcb_args, {f})" for f, _ in N.GcbArgs._fields_)
        + "".join(f"P(rbf_gcb_state, {f})" for f, _ in N.GcbState._fields_)
        + "".join(f"P(rbf_gcb_record, {f})" for f, _ in N.GcbRecord._fields_)
        + "return 0;}\n"
    )
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", str(REPO / "include"), str(src), "-o", str(exe)], check=True)
    lines = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = dict(line.split() for line in lines if line)
    assert int(got["rbf_gcb_args"]) == ctypes.sizeof(N.GcbArgs)
    assert int(got["rbf_gcb_state"]) == ctypes.sizeof(N.GcbState)
    assert int(got["rbf_gcb_record"]) == ctypes.sizeof(N.GcbRecord)
    for cls, cname in ((N.GcbArgs, "rbf_gcb_args"), (N.GcbState, "rbf_gcb_state"),
                       (N.GcbRecord, "rbf_gcb_record")):
        for f, _ in cls._fields_:
            assert int(got[f"{cname}.{f}"]) == getattr(cls, f).offset, (cname, f)


def test_scratch_size_queries_need_no_gpu():
    lib = N.load()
    assert lib.rbf_errors_scratch_bytes(1000) >= 256
    assert lib.rbf_chol_scratch_bytes(100) >= 4 * 800
    assert lib.rbf_gcb_scratch_bytes(20000, 512, 148) > 20000 * 8

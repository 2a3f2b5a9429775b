"""Stage the reference's own unit tests as a drop-in conformance suite.

    python tools/conformance/stage.py            # in the build container

Copies (does not commit: ``build/`` is git-ignored but travels to the GPU box
with the repo snapshot) the reference's test files for the hot-path modules --
``tests/test_core.py``, ``test_selection.py``, ``test_estimator.py``, plus
``test_metrics.py``, ``test_meshio.py``, ``test_cli.py`` and ``test_deformers.py``
for the §8(f) rows -- and its ``conftest.py`` into ``build/conformance/``, with:

* ``build/conformance/rbfdeform/__init__.py`` = tools/conformance/rbfdeform_shim.py
  (the alias of ``rbfdeform`` to this package);
* ``build/conformance/rbfdeform/synthetic.py`` = the reference's own desk-wing
  generator (a test fixture outside the hot path; also registered as the CLI's
  ``make-wing``);
* ``build/conformance/SOURCE`` recording where the files came from.

tests/test_gpu_conformance.py runs the staged suite on the B200 (``-m gpu``) and
checks every failure against ``KNOWN`` there; /root/reference is never read on
the GPU box.
"""

import hashlib
import shutil
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[2]
REF = Path("/root/reference/pkg")
OUT = REPO / "build" / "conformance"
TESTS = ["conftest.py", "test_core.py", "test_selection.py", "test_estimator.py", "test_metrics.py",
         "test_meshio.py", "test_cli.py", "test_deformers.py"]
FIXTURES = ["synthetic.py"]


def main():
    if not (REF / "tests" / "test_core.py").exists():
        print("reference tests not found at", REF, file=sys.stderr)
        return 1
    if OUT.exists():
        shutil.rmtree(OUT)
    (OUT / "rbfdeform").mkdir(parents=True)
    lines = []
    for name in TESTS:
        src = REF / "tests" / name
        shutil.copyfile(src, OUT / name)
        lines.append(f"{src} sha256={hashlib.sha256(src.read_bytes()).hexdigest()}")
    for name in FIXTURES:
        src = REF / "src" / "rbfdeform" / name
        shutil.copyfile(src, OUT / "rbfdeform" / name)
        lines.append(f"{src} sha256={hashlib.sha256(src.read_bytes()).hexdigest()}")
    src = REF / "src" / "rbfdeform" / "metrics.py"  # cell_quality / quality_report only
    shutil.copyfile(src, OUT / "rbfdeform" / "_ref_metrics.py")
    lines.append(f"{src} sha256={hashlib.sha256(src.read_bytes()).hexdigest()}")
    shutil.copyfile(Path(__file__).with_name("rbfdeform_shim.py"), OUT / "rbfdeform" / "__init__.py")
    (OUT / "pytest.ini").write_text("[pytest]\naddopts = -p no:cacheprovider\n")
    (OUT / "SOURCE").write_text("\n".join(lines) + "\n")
    print("staged", len(TESTS), "test files and", len(FIXTURES), "fixtures into", OUT)
    return 0


if __name__ == "__main__":
    sys.exit(main())

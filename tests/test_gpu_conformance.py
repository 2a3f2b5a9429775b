"""The reference's own unit tests, run against this package as the drop-in
conformance suite: test_core.py, test_selection.py,
test_estimator.py, test_metrics.py and test_meshio.py from the reference, with
``rbfdeform`` aliased to ``paper_2004_04817_b200``
(tools/conformance/rbfdeform_shim.py). The files are staged by
``python tools/conformance/stage.py`` into the git-ignored ``build/conformance``
(reference sources are not committed); the staged copy travels to the GPU box
with the repository snapshot. Skipped when not staged.

Every failure must be listed in KNOWN with its reason."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
REPO = Path(__file__).resolve().parent.parent
STAGED = REPO / "build" / "conformance"

# test node id -> why it differs from the reference (none so far)
KNOWN = {}


def test_reference_unit_tests_pass_through_alias(cuda, tmp_path):
    if not (STAGED / "test_core.py").exists():
        pytest.skip("conformance suite not staged (python tools/conformance/stage.py)")
    report = tmp_path / "report.xml"
    env = dict(os.environ, PYTHONPATH=str(REPO), PYTHONDONTWRITEBYTECODE="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                        f"--junitxml={report}", "."], cwd=STAGED, env=env, capture_output=True,
                       text=True, timeout=1800)
    import xml.etree.ElementTree as ET

    root = ET.parse(report).getroot()
    cases, failed = 0, {}
    for tc in root.iter("testcase"):
        cases += 1
        bad = tc.find("failure") if tc.find("failure") is not None else tc.find("error")
        if bad is not None:
            failed[f"{tc.get('classname')}::{tc.get('name')}"] = (bad.get("message") or "")[:300]
    out = REPO / "gpurun_out"
    if out.is_dir():
        (out / "conformance_report.json").write_text(json.dumps(
            {"cases": cases, "failed": failed, "tail": r.stdout[-3000:]}, indent=1))
    assert cases >= 150, r.stdout[-2000:]
    unexpected = {k: v for k, v in failed.items() if k not in KNOWN}
    assert not unexpected, json.dumps(unexpected, indent=1)

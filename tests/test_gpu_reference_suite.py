"""The reference's own 148-test suite (tests/reference_suite, vendored from
/root/reference/pkg/tests) run against the drop-in: ``import memplan``
resolves to paper_1903_06631_b200 (tests/reference_suite/_alias), so every
call goes through the device library.  A child pytest keeps its
``conftest``/``oracles`` modules apart from ours.

EXPECTED_FAILURES lists any reference test the drop-in does not pass, each
with the reason; every other test must pass.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SUITE = os.path.join(HERE, "reference_suite")

EXPECTED_FAILURES: dict[str, str] = {}


def test_reference_suite_passes_against_dropin(tmp_path):
    report = tmp_path / "report.jsonl"
    plugin = tmp_path / "record_outcomes.py"
    plugin.write_text(
        "import json, os\n"
        "def pytest_runtest_logreport(report):\n"
        "    if report.when == 'call' or report.outcome != 'passed':\n"
        "        with open(os.environ['MP_SUITE_REPORT'], 'a') as fh:\n"
        "            fh.write(json.dumps([report.nodeid, report.when, report.outcome,\n"
        "                                 str(report.longrepr)[-1500:] if report.failed else '']) + '\\n')\n")
    env = dict(os.environ, MP_SUITE_REPORT=str(report),
               PYTHONPATH=os.pathsep.join([os.path.join(SUITE, "_alias"), ROOT, str(tmp_path),
                                           os.environ.get("PYTHONPATH", "")]))
    p = subprocess.run([sys.executable, "-m", "pytest", SUITE, "-q", "-p", "record_outcomes", "-p",
                        "no:cacheprovider", "--rootdir", SUITE, "-o", "addopts="],
                       capture_output=True, text=True, timeout=1500, env=env, cwd=SUITE)
    rows = [json.loads(ln) for ln in report.read_text().splitlines()] if report.exists() else []
    out = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(out):
        with open(os.path.join(out, "reference_suite.jsonl"), "w") as fh:
            fh.write("\n".join(json.dumps(r) for r in rows) + "\n")
    calls = [r for r in rows if r[1] == "call"]
    failed = {r[0]: r[3] for r in rows if r[2] == "failed"}
    unexpected = {k: v for k, v in failed.items() if k.split("::", 1)[-1] not in EXPECTED_FAILURES}
    assert len(calls) >= 148, (len(calls), p.stdout[-3000:], p.stderr[-3000:])
    assert not unexpected, json.dumps(unexpected, indent=1)[:8000]

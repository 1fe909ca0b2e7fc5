"""The command line (paper_1903_06631_b200.cli) replays the reference CLI's
recorded sessions (tests/golden/cli.json.gz, make_golden_cli.py): identical
exit codes, stdout, stderr and report files, byte for byte."""
import json  # noqa: F401
import os
import subprocess
import sys

import pytest

from golden_util import load  # noqa: F401

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sessions():
    import gzip
    with gzip.open(os.path.join(ROOT, "tests", "golden", "cli.json.gz"), "rt") as fh:
        return json.load(fh)["sessions"]


SESSIONS = _sessions()


@pytest.mark.parametrize("si", range(len(SESSIONS)))
def test_cli_replays_reference_session(si, tmp_path):
    sess = SESSIONS[si]
    env = dict(os.environ, PYTHONPATH=ROOT)
    env.pop("MEMPLAN_SEED", None)
    env.update(sess["env"])
    for step in sess["steps"]:
        if "write" in step:
            name, text = step["write"]
            (tmp_path / name).write_text(text)
            continue
        r = subprocess.run([sys.executable, "-m", "paper_1903_06631_b200", *step["args"]], cwd=tmp_path, env=env,
                           capture_output=True, text=True)
        assert (r.returncode, r.stdout, r.stderr) == (step["rc"], step["stdout"], step["stderr"]), step["args"]
    files = {}
    for root, _dirs, names in os.walk(tmp_path):
        for nm in names:
            p = os.path.join(root, nm)
            with open(p, encoding="utf-8") as fh:
                files[os.path.relpath(p, tmp_path)] = fh.read()
    assert sorted(files) == sorted(sess["files"])
    for name, text in sess["files"].items():
        assert files[name] == text, name

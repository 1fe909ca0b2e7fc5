"""Golden CLI transcripts, produced by the REFERENCE command line.

Run in the build container only:  python tests/golden/make_golden_cli.py

Each session runs ``python -m memplan <args>`` (the reference, from
/root/reference/pkg/src) in a fresh directory and records the exit code,
stdout, stderr and every file the commands wrote; tests/test_gpu_cli.py
replays the same commands with ``python -m paper_1903_06631_b200`` and
requires identical bytes.
"""
from __future__ import annotations

import gzip
import json
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"


def limits_for(path, fracs):
    sys.path.insert(0, REF)
    import memplan as mp
    pf = mp.IterationAnalyzer().fit(mp.load_trace(path)).profile_
    return ",".join(str(int(pf.load.peak_bytes * f)) for f in fracs)


def session(cmds, env_extra=None):
    with tempfile.TemporaryDirectory() as d:
        out = []
        for args in cmds:
            if callable(args):
                args = args(d)
            if args and args[0] == "@write":
                with open(os.path.join(d, args[1]), "w") as fh:
                    fh.write(args[2])
                out.append({"write": args[1:]})
                continue
            env = dict(os.environ, PYTHONPATH=REF, **(env_extra or {}))
            env.pop("MEMPLAN_SEED", None) if not env_extra else None
            r = subprocess.run([sys.executable, "-m", "memplan", *args], cwd=d, env=env, capture_output=True,
                               text=True)
            out.append({"args": args, "rc": r.returncode, "stdout": r.stdout, "stderr": r.stderr})
        files = {}
        for root, _dirs, names in os.walk(d):
            for nm in names:
                p = os.path.join(root, nm)
                with open(p, encoding="utf-8") as fh:
                    files[os.path.relpath(p, d)] = fh.read()
        return {"steps": out, "files": files, "env": env_extra or {}}


def main():
    sessions = []
    sessions.append(session([
        ["gen", "--out", "t.jsonl", "--layers", "5", "--iterations", "4", "--scale", "0.25", "--seed", "3"],
        ["gen", "--out", "t.csv", "--layers", "4", "--format", "csv", "--seed", "1"],
        ["analyze", "--trace", "t.jsonl", "--out-dir", "a"],
        ["plan", "--trace", "t.jsonl", "--out-dir", "p1"],
        ["plan", "--trace", "t.csv", "--policy", "first_fit", "--out-dir", "p2"],
        lambda d: ["swap", "--trace", "t.jsonl", "--limit", limits_for(os.path.join(d, "t.jsonl"), (0.95, 0.85)),
                   "--out-dir", "s1"],
        lambda d: ["full", "--trace", "t.jsonl", "--limit", limits_for(os.path.join(d, "t.jsonl"), (0.9,)),
                   "--score", "bo", "--bo-budget", "6", "--bandwidth", "2e9", "--out-dir", "f1"],
        lambda d: ["swap", "--trace", "t.csv", "--limit", limits_for(os.path.join(d, "t.csv"), (0.92,)),
                   "--score", "aoa", "--threshold", "1MiB", "--out-dir", "s2"],
        ["swap", "--trace", "t.jsonl", "--limit", "1"],
        ["swap", "--trace", "t.jsonl", "--limit", "5,10"],
        ["plan", "--trace", "missing.jsonl"],
        ["@write", "cfg.json", json.dumps({"policy": "first_fit", "out_dir": "pc"})],
        ["plan", "--trace", "t.jsonl", "--config", "cfg.json"],
        ["plan", "--trace", "t.jsonl", "--config", "cfg.json", "--policy", "best_fit"],
    ]))
    sessions.append(session([["gen", "--out", "e.jsonl", "--layers", "3", "--seed", "5"],
                             ["analyze", "--trace", "e.jsonl"]], env_extra={"MEMPLAN_SEED": "11"}))
    with gzip.open(os.path.join(HERE, "cli.json.gz"), "wt") as fh:
        json.dump({"sessions": sessions, "python": sys.version}, fh)
    print(sum(len(s["steps"]) for s in sessions), "steps,", sum(len(s["files"]) for s in sessions), "files")


if __name__ == "__main__":
    main()

"""``import memplan`` resolves to the B200 drop-in (paper_1903_06631_b200).

Put this directory first on PYTHONPATH to run the reference's own test
suite (tests/reference_suite, vendored from the reference's pkg/tests)
against the drop-in: ``memplan`` and every ``memplan.<submodule>`` name the
reference package has become the drop-in's modules.
"""
import importlib
import sys

_pkg = importlib.import_module("paper_1903_06631_b200")
for _sub in ("autoswap", "bo", "cli", "errors", "estimators", "iteration", "smartpool", "swapsim", "synth",
             "trace", "validation"):
    sys.modules[f"{__name__}.{_sub}"] = importlib.import_module(f"paper_1903_06631_b200.{_sub}")
sys.modules[__name__] = _pkg

"""pytest plugin for the reference-suite replay (tests/test_reference_suite_gpu.py).

Loaded with ``-p dropin_plugin`` before the reference's own test modules are
collected: it swaps ``chainscan.chained_scan`` — in the package namespace,
in ``chainscan.chained`` and in ``chainscan.bench`` (whose ``run_algorithm``
dispatches "chained" to it, bench.py:121-147) — for the GPU drop-in
``paper_1604_04815_b200.chained_scan``, and ``chainscan.cli.main`` for the
drop-in's chainscan-compatible command line.  The test modules then import the
swapped function (``from chainscan import chained_scan``) and run unchanged,
with the reference's real ``ScanProblem``, ``make_operator`` and
``ChainConfig`` objects and its exception classes.  At the end it writes how
many scans went through the drop-in and how many native kernels launched,
so the caller can prove the device path ran.
"""

import json
import os

import chainscan
import chainscan.bench
import chainscan.chained
import chainscan.cli

import paper_1604_04815_b200 as P
from paper_1604_04815_b200 import _native

_calls = {"dropin": 0, "nonempty": 0}


def _dropin(problem, config=None):
    _calls["dropin"] += 1
    _calls["nonempty"] += 1 if problem.x.size else 0
    return P.chained_scan(problem, config)


for _mod in (chainscan, chainscan.chained, chainscan.bench):
    _mod.chained_scan = _dropin

# the command line: chainscan's CLI tests call chainscan.cli.main(argv); the
# drop-in's front end (python -m paper_1604_04815_b200) takes its place
from paper_1604_04815_b200 import cli as _cli  # noqa: E402

chainscan.cli.main = _cli.main


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("REFSUITE_REPORT")
    if path:
        with open(path, "w") as f:
            json.dump({"dropin_calls": _calls["dropin"], "nonempty_calls": _calls["nonempty"],
                       "native_launches": _native.launch_count()}, f)

"""Drop-in compatibility with the reference's own objects, on CPU (no device
call is reached): the reference's ``ScanProblem`` / ``make_operator`` /
``ChainConfig`` are accepted, and every error the drop-in raises is caught
by the reference's exception classes (reference.py:34-35, operators.py:34-35,
chained.py:48-53) as well as by this package's.

Uses the reference package staged by ``oracle/stage_reference.py`` (test
infrastructure); skipped when it is not staged."""

import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SRC = os.path.join(REPO, "oracle", "_ref", "pkg", "src")


@pytest.fixture(scope="module")
def chainscan():
    if not os.path.isdir(os.path.join(REF_SRC, "chainscan")):
        pytest.skip("reference not staged (oracle/stage_reference.py)")
    sys.path.insert(0, REF_SRC)
    try:
        import chainscan as cs
        yield cs
    finally:
        sys.path.remove(REF_SRC)


def test_errors_are_reference_classes(chainscan):
    import paper_1604_04815_b200 as P
    x = np.arange(10, dtype=np.int32)
    # dtype mismatch between x and the operator -> ShapeError
    with pytest.raises(chainscan.ShapeError) as ei:
        P.chained_scan(chainscan.ScanProblem(x, chainscan.make_operator("add", "i64")))
    assert isinstance(ei.value, P.ShapeError)
    # an operator the device does not implement -> UnsupportedOperatorError
    class Mul:
        name, dtype, identity = "mul", np.dtype(np.int32), np.int32(1)
    with pytest.raises(chainscan.UnsupportedOperatorError) as ei:
        P.chained_scan(chainscan.ScanProblem(x, Mul()))
    assert isinstance(ei.value, P.UnsupportedOperatorError)
    # this package's own factory and problem raise them too
    with pytest.raises(chainscan.UnsupportedOperatorError):
        P.make_operator("xor", "i32")
    with pytest.raises(chainscan.ShapeError):
        P.ScanProblem(np.zeros((2, 2), dtype=np.int32), P.make_operator("add", "i32"))


def test_status_codes_map_to_reference_classes(chainscan):
    from paper_1604_04815_b200 import _native as N
    from paper_1604_04815_b200.errors import raise_for_status
    cases = {N.LS_ERR_INVALID_ARG: chainscan.ShapeError, N.LS_ERR_UNSUPPORTED_DTYPE: chainscan.UnsupportedOperatorError,
             N.LS_ERR_LIVENESS: chainscan.LivenessError, N.LS_ERR_PROTOCOL: chainscan.ProtocolViolation}
    for code, cls in cases.items():
        with pytest.raises(cls):
            raise_for_status(code)


def test_reference_objects_accepted_up_to_the_device(chainscan):
    import paper_1604_04815_b200 as P
    op = chainscan.make_operator("add", "f32")
    # empty input returns the output untouched without touching the device
    out = np.empty(0, dtype=np.float32)
    got = P.chained_scan(chainscan.ScanProblem(np.empty(0, dtype=np.float32), op, out=out),
                         chainscan.ChainConfig(b=1))
    assert got is out
    # on_block (a host callback per block) is refused with a clear error
    with pytest.raises(ValueError, match="on_block"):
        P.chained_scan(chainscan.ScanProblem(np.ones(4, dtype=np.float32), op),
                       chainscan.ChainConfig(b=2, on_block=lambda w, b: None))
